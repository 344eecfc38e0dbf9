// sl.cuh -- semi-Lagrangian gather kernels: RK2 departure points (Eq. 6) and the
// tricubic interpolation at those points (reading A6: tensor cubic Lagrange on the
// 4x4x4 nodes q-1..q+2 with periodic wrap) fused with the epilogue of each transport step
// (state, adjoint, incremental state / adjoint: Eq. 7, Algorithm 2).
//
// Layout and plan.  Output tiles are TX x TY x TZ = 32 x 8 x 8 voxels (one 256-thread CTA; lane =
// x1, warp = x2, each thread walks TZ points along x3).  Because departure points move with the
// (stationary) velocity, the input box a tile reads is fixed once per velocity and direction:
// the plan kernel (the analogue of the paper's "interpolation planner") stores per tile the
// box origin (min floor(s) - 1, unwrapped) and extents.  Each transport step then stages that box
// from L2/HBM into shared memory with coalesced row loads (periodic wrap on the fly) and gathers all
// 64 stencil values from shared memory.  Tiles whose box exceeds the shared-memory capacity chosen
// for the launch fall back to gathering straight from global memory (same arithmetic).
#pragma once
#include "common.cuh"

namespace dr {

constexpr int SL_TX = 32, SL_TY = 8, SL_TZ = 4, SL_THREADS = SL_TX * SL_TY;
constexpr int PLAN_INTS = 8;  // ox, oy, oz, ex, ey, ez, pad, pad

// Lagrange weights for nodes -1, 0, 1, 2 at t in [0, 1) (reading A6)
// (factored: a = t(t-1), b = (t+1)(t-2) = a - 2; w_-1 = a (2-t)/6, w_0 = b (t-1)/2, w_1 = -b t/2, w_2 = a (t+1)/6)
template <typename T>
__device__ __forceinline__ void lagrange4(T t, T w[4]) {
    const T sixth = T(1) / T(6);
    const T a = t * (t - T(1));
    const T b = a - T(2);
    w[0] = a * (T(2) * sixth - t * sixth);
    w[1] = b * (T(0.5) * t - T(0.5));
    w[2] = b * (T(-0.5) * t);
    w[3] = a * (t * sixth + sixth);
}

template <typename T>
__device__ __forceinline__ T floor_t(T x);
template <>
__device__ __forceinline__ float floor_t<float>(float x) { return floorf(x); }
template <>
__device__ __forceinline__ double floor_t<double>(double x) { return floor(x); }

// Departure point of node i with displacement d (cells): s = i - d, q = i + floor(-d), t = -d - floor(-d)
// (exact in floating point: subtracting the integer floor(-d) from -d loses nothing).
template <typename T>
__device__ __forceinline__ void cell_of(int i, T d, int& q, T& t) {
    const T e = -d;
    const T fl = floor_t(e);
    t = e - fl;
    q = i + (int)fl;
}

template <typename T>
__device__ __forceinline__ T interp_smem(const T* __restrict__ b, int sy, int sz, const T w1[4], const T w2[4],
                                         const T w3[4]) {
    T acc = T(0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        T accb = T(0);
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const T* r = b + c * sz + bb * sy;
            const T row = w1[0] * r[0] + w1[1] * r[1] + w1[2] * r[2] + w1[3] * r[3];
            accb += w2[bb] * row;
        }
        acc += w3[c] * accb;
    }
    return acc;
}

template <typename T>
__device__ __forceinline__ T interp_global(const T* __restrict__ f, const Grid& g, int q1, int q2, int q3,
                                           const T w1[4], const T w2[4], const T w3[4]) {
    T acc = T(0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int j3 = wrapi(q3 + c - 1, g.n3);
        T accb = T(0);
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const int j2 = wrapi(q2 + bb - 1, g.n2);
            const T* r = f + ((int64_t)j3 * g.n2 + j2) * g.n1;
            T row = T(0);
#pragma unroll
            for (int a = 0; a < 4; ++a) row += w1[a] * __ldg(r + wrapi(q1 + a - 1, g.n1));
            accb += w2[bb] * row;
        }
        acc += w3[c] * accb;
    }
    return acc;
}

__device__ __forceinline__ void tile_coords(const Grid& g, int tile, int& x0, int& y0, int& z0) {
    const int ntx = (g.n1 + SL_TX - 1) / SL_TX, nty = (g.n2 + SL_TY - 1) / SL_TY;
    x0 = (tile % ntx) * SL_TX;
    y0 = ((tile / ntx) % nty) * SL_TY;
    z0 = (tile / (ntx * nty)) * SL_TZ;
}

// ---------------------------------------------------------------------------------------------
// Plan: per tile, the unwrapped box [min q - 1, max q + 2] of the stencil nodes of its departure
// points, and the running maximum extents over all tiles (for sizing shared memory).
template <typename T>
__global__ void __launch_bounds__(SL_THREADS) k_sl_plan(Grid g, const T* __restrict__ d, int* __restrict__ plan,
                                                        int* __restrict__ maxext) {
    __shared__ int red[6];
    if (threadIdx.x < 6) red[threadIdx.x] = (threadIdx.x < 3) ? INT_MAX : INT_MIN;
    __syncthreads();
    int x0, y0, z0;
    tile_coords(g, blockIdx.x, x0, y0, z0);
    const int x = x0 + (threadIdx.x % SL_TX), y = y0 + threadIdx.x / SL_TX;
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
    if (x < g.n1 && y < g.n2) {
        for (int k = 0; k < SL_TZ; ++k) {
            const int z = z0 + k;
            if (z >= g.n3) break;
            const int64_t id = ((int64_t)z * g.n2 + y) * g.n1 + x;
            const int ii[3] = {x, y, z};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                int q;
                T t;
                cell_of<T>(ii[a], d[a * g.M + id], q, t);
                mn[a] = min(mn[a], q);
                mx[a] = max(mx[a], q);
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(&red[a], mn[a]);
            atomicMax(&red[3 + a], mx[a]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int* p = plan + (int64_t)blockIdx.x * PLAN_INTS;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            p[a] = red[a] - 1;
            p[3 + a] = red[3 + a] - red[a] + 4;
            atomicMax(&maxext[a], p[3 + a]);
        }
        p[6] = p[7] = 0;
    }
}

// ---------------------------------------------------------------------------------------------
// Epilogues of the fused gather kernel.  `load(id)` fetches (and pre-reduces) the voxel's pointwise
// operands before the box wait, so their latency overlaps the shared-memory staging; `store(id, val,
// pre)` finishes the step with the NC interpolated components `val` at the departure point.
template <typename T>
struct EpiStore {  // state solve: rho_{j+1} = I[rho_j](X+)   (Eq. 7 with f = 0)
    T* out;
    struct Pre {};
    __device__ __forceinline__ Pre load(int64_t) const { return Pre{}; }
    __device__ __forceinline__ void store(int64_t id, const T* val, const Pre&) const { out[id] = val[0]; }
};

template <typename T>
struct EpiAdjoint {  // adjoint-like step: nu_{k-1} = scale * m * I[nu_k](X-)  (Eq. 7, f = nu div v; D7)
    T* out;
    const T* m;  // nullable (isochoric: m == 1)
    T scale;
    struct Pre { T m; };
    __device__ __forceinline__ Pre load(int64_t id) const { return Pre{m ? scale * __ldg(m + id) : scale}; }
    __device__ __forceinline__ void store(int64_t id, const T* val, const Pre& p) const { out[id] = p.m * val[0]; }
};

template <typename T>
struct EpiIncState {  // Algorithm 2 with the merged gather: g_{j+1} = I[g_j](X+) + c f_{j+1}, f = -vt.G_{j+1}
    T* out;
    const T* vt;  // vector field
    const T* G;   // vector field grad rho_{j+1}
    T c;
    int64_t M;
    struct Pre { T cf; };
    __device__ __forceinline__ Pre load(int64_t id) const {
        const T f = -(__ldg(vt + id) * __ldg(G + id) + __ldg(vt + M + id) * __ldg(G + M + id) +
                      __ldg(vt + 2 * M + id) * __ldg(G + 2 * M + id));
        return Pre{c * f};
    }
    __device__ __forceinline__ void store(int64_t id, const T* val, const Pre& p) const { out[id] = val[0] + p.cf; }
};

template <typename T>
struct EpiMultiplier {  // m = 1 + dt/2 (Dbar + D + dt Dbar D), Dbar = I[div v](X-)  (D7)
    T* m;
    const T* D;
    T dt;
    struct Pre { T D; };
    __device__ __forceinline__ Pre load(int64_t id) const { return Pre{__ldg(D + id)}; }
    __device__ __forceinline__ void store(int64_t id, const T* val, const Pre& p) const {
        const T Db = val[0];
        m[id] = T(1) + T(0.5) * dt * (Db + p.D + dt * Db * p.D);
    }
};

template <typename T>
struct EpiDeparture {  // d = sigma dt/2 (v(x) + I[v](X*)) / h  (Eq. 6, cell units)
    T* d;
    const T* v;
    T c[3];  // sigma * dt / (2 h_a)
    int64_t M;
    struct Pre { T v[3]; };
    __device__ __forceinline__ Pre load(int64_t id) const {
        return Pre{{__ldg(v + id), __ldg(v + M + id), __ldg(v + 2 * M + id)}};
    }
    __device__ __forceinline__ void store(int64_t id, const T* val, const Pre& p) const {
#pragma unroll
        for (int a = 0; a < 3; ++a) d[a * M + id] = c[a] * (p.v[a] + val[a]);
    }
};

template <typename T, int NC>
struct Src {
    const T* p[NC];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Shared-memory box geometry per (value type, components): compile-time strides so every one of the
// 64 stencil loads is an LDS with an immediate offset from one per-point base address.  BX is a
// multiple of 32 words so that lanes of a warp whose departure rows differ stay on distinct banks.
template <typename T, int NC>
struct BoxGeom;
template <> struct BoxGeom<float, 1> { static constexpr int BX = 64, BY = 16, BZ = 12; };   //  48 KB
template <> struct BoxGeom<float, 3> { static constexpr int BX = 64, BY = 16, BZ = 16; };   // 192 KB
template <> struct BoxGeom<double, 1> { static constexpr int BX = 64, BY = 16, BZ = 16; };  // 128 KB
template <> struct BoxGeom<double, 3> { static constexpr int BX = 32, BY = 12, BZ = 12; };  // 108 KB

template <typename T, int NC>
constexpr size_t box_bytes() {
    return (size_t)NC * BoxGeom<T, NC>::BX * BoxGeom<T, NC>::BY * BoxGeom<T, NC>::BZ * sizeof(T);
}

template <typename T, int BX, int BY>
__device__ __forceinline__ T interp_box(const T* __restrict__ b, const T w1[4], const T w2[4], const T w3[4]) {
    T acc = T(0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        T accb = T(0);
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const T* r = b + (c * BY + bb) * BX;
            const T row = w1[0] * r[0] + w1[1] * r[1] + w1[2] * r[2] + w1[3] * r[3];
            accb += w2[bb] * row;
        }
        acc += w3[c] * accb;
    }
    return acc;
}

// Fused gather + epilogue.  Grid: one CTA per tile.  Dynamic smem: box_bytes<T, NC>().
// Phases: (A) stage the tile's box with 16-byte cp.async (periodic wrap per chunk; x origin aligned
// down to VEC = 16 B / sizeof(T), which never straddles the wrap since N1 is a multiple of VEC);
// (B) meanwhile load the displacements and the epilogue operands of the thread's 8 points; (C) wait
// + barrier; (D) gather the 64 stencil values per point from shared memory and finish the step.
// Tiles whose box exceeds the compile-time capacity gather from global memory instead.
template <typename T, int NC, class Epi>
__global__ void __launch_bounds__(SL_THREADS, (sizeof(T) == 4 && NC == 1) ? 4 : 1) k_sl_gather(Grid g, Src<T, NC> src, const T* __restrict__ d,
                                                          const int* __restrict__ plan, Epi epi) {
    constexpr int VEC = 16 / (int)sizeof(T);
    constexpr int BX = BoxGeom<T, NC>::BX, BY = BoxGeom<T, NC>::BY, BZ = BoxGeom<T, NC>::BZ;
    constexpr int SC = BX * BY * BZ;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* box = reinterpret_cast<T*>(smem_raw);
    int x0, y0, z0;
    tile_coords(g, blockIdx.x, x0, y0, z0);
    const int* pl = plan + (int64_t)blockIdx.x * PLAN_INTS;
    const int ox = pl[0] & ~(VEC - 1), oy = pl[1], oz = pl[2];
    const int ex = ((pl[0] + pl[3] - ox) + VEC - 1) & ~(VEC - 1), ey = pl[4], ez = pl[5];
    const bool fits = ex <= BX && ey <= BY && ez <= BZ;
    const int lane = threadIdx.x % SL_TX, wy = threadIdx.x / SL_TX;
    const int x = x0 + lane, y = y0 + wy;
    const bool xyok = x < g.n1 && y < g.n2;

    // (A) asynchronous staging of the box: thread -> fixed 16-byte chunk column, rows strided by
    // SL_THREADS / NCHP (no divisions in the loop)
    if (fits) {
        constexpr int NCHP = BX / VEC;              // chunk columns of a full-width row (power of two)
        constexpr int RSTEP = SL_THREADS / NCHP;
        const int nch = ex / VEC;
        const int ch = threadIdx.x % NCHP;
        if (ch < nch) {
            int yy = threadIdx.x / NCHP, zz = 0;
            while (yy >= ey) { yy -= ey; ++zz; }
            while (zz < ez) {
                const int gy = wrapi(oy + yy, g.n2), gz = wrapi(oz + zz, g.n3);
                const int64_t gofs = ((int64_t)gz * g.n2 + gy) * g.n1 + wrapi(ox + ch * VEC, g.n1);
                T* dst = box + (zz * BY + yy) * BX + ch * VEC;
#pragma unroll
                for (int c = 0; c < NC; ++c) cp_async16(dst + c * SC, src.p[c] + gofs);
                yy += RSTEP;
                while (yy >= ey) { yy -= ey; ++zz; }
            }
        }
    }

    // (B) displacements and epilogue operands of this thread's points
    T dd[SL_TZ][3];
    typename Epi::Pre pre[SL_TZ];
#pragma unroll
    for (int k = 0; k < SL_TZ; ++k) {
        const int z = z0 + k;
        const int64_t id = ((int64_t)z * g.n2 + y) * g.n1 + x;
        const bool ok = xyok && z < g.n3;
#pragma unroll
        for (int a = 0; a < 3; ++a) dd[k][a] = ok ? __ldg(d + a * g.M + id) : T(0);
        if (ok) pre[k] = epi.load(id);
    }

    // (C)
    if (fits) cp_async_wait_all();
    __syncthreads();
    if (!xyok) return;
    const int kmax = min(SL_TZ, g.n3 - z0);

    // (D)
    if (fits) {
#pragma unroll
        for (int k = 0; k < SL_TZ; ++k) {
            if (k >= kmax) break;
            const int z = z0 + k;
            int q1, q2, q3;
            T t1, t2, t3;
            cell_of<T>(x, dd[k][0], q1, t1);
            cell_of<T>(y, dd[k][1], q2, t2);
            cell_of<T>(z, dd[k][2], q3, t3);
            T w1[4], w2[4], w3[4];
            lagrange4(t1, w1);
            lagrange4(t2, w2);
            lagrange4(t3, w3);
            const T* b = box + ((q3 - 1 - oz) * BY + (q2 - 1 - oy)) * BX + (q1 - 1 - ox);
            T val[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) val[c] = interp_box<T, BX, BY>(b + c * SC, w1, w2, w3);
            epi.store(((int64_t)z * g.n2 + y) * g.n1 + x, val, pre[k]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < SL_TZ; ++k) {
            if (k >= kmax) break;
            const int z = z0 + k;
            int q1, q2, q3;
            T t1, t2, t3;
            cell_of<T>(x, dd[k][0], q1, t1);
            cell_of<T>(y, dd[k][1], q2, t2);
            cell_of<T>(z, dd[k][2], q3, t3);
            T w1[4], w2[4], w3[4];
            lagrange4(t1, w1);
            lagrange4(t2, w2);
            lagrange4(t3, w3);
            T val[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) val[c] = interp_global(src.p[c], g, q1, q2, q3, w1, w2, w3);
            epi.store(((int64_t)z * g.n2 + y) * g.n1 + x, val, pre[k]);
        }
    }
}

// First-stage displacement of Eq. 6: d* = sigma dt v / h (cells), X* = x - h d*.
template <typename T>
__global__ void k_dstar(Grid g, const T* __restrict__ v, T* __restrict__ dstar, T c0, T c1, T c2) {
    const int64_t n = 3 * g.M;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(e / g.M);
        const T c = a == 0 ? c0 : (a == 1 ? c1 : c2);
        dstar[e] = c * v[e];
    }
}

// Interpolation at arbitrary points (test hook dr_op_interp): s in cell coordinates.
template <typename T>
__global__ void k_interp_points(Grid g, const T* __restrict__ f, int64_t npts, const T* __restrict__ s,
                                T* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts; p += (int64_t)gridDim.x * blockDim.x) {
        T w[3][4];
        int q[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const T sa = s[a * npts + p];
            const T fl = floor_t(sa);
            q[a] = (int)fl;
            lagrange4(sa - fl, w[a]);
        }
        out[p] = interp_global(f, g, q[0], q[1], q[2], w[0], w[1], w[2]);
    }
}

}  // namespace dr
