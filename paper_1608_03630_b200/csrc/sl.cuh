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
#include "fft.cuh"  // mbarrier / bulk-copy helpers (the TMA box staging)

namespace dr {

// A warp is one x1 row of the tile (lane = x1).  SL_TX <= 32 columns per tile: with 31 (DR_TX=31) the
// 32 lanes' stencil columns never span 33 words, so the two end lanes of a warp whose departure floor
// steps up along x1 cannot collide in one bank (tools/bank_sim.py: 1.30 -> 1.05 wavefronts per LDS);
// lane 31 idles.
#ifndef DR_TX
#define DR_TX 32
#endif
constexpr int SL_TX = DR_TX, SL_LANES = 32, SL_TY = 8, SL_TZ = 8, SL_THREADS = SL_LANES * SL_TY;
static_assert(SL_TX <= SL_LANES, "tile width");
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
        const int j3 = g.ghost ? q3 + c - 1 - g.z0 + g.zg : wrap2(q3 + c - 1, g.n3);
        DR_ASSERT(j3 >= 0 && j3 < g.n3 + g.zg + g.zgh);
        T accb = T(0);
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const int j2 = wrap2(q2 + bb - 1, g.n2);
            const T* r = f + ((int64_t)j3 * g.n2 + j2) * g.n1;
            T row = T(0);
#pragma unroll
            for (int a = 0; a < 4; ++a) row += w1[a] * __ldg(r + wrap2(q1 + a - 1, g.n1));
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
// maxext[0..2]: running maximum box extents; maxext[3] is set to 1 when, in slab mode, a tile's box
// leaves the rank's planes plus ghosts (the displacement exceeds the ghost width: DR_ERR_PLAN).
// DSTAR: d is written here, d_a = c_a v_a (the first-stage displacement of Eq. 6, c_a = sigma dt / h_a),
// while its plan is taken -- one pass over v instead of a separate d pass and a plan pass over d.
template <typename T>
struct DstarIn {
    const T* v[3];
    T c[3];
};
template <typename T, bool DSTAR = false>
__global__ void __launch_bounds__(SL_THREADS) k_sl_plan(Grid g, const T* __restrict__ d_in, int* __restrict__ plan,
                                                        int* __restrict__ maxext, DstarIn<T> ds = DstarIn<T>{}) {
    T* d = const_cast<T*>(d_in);
    __shared__ int red[6];
    if (threadIdx.x < 6) red[threadIdx.x] = (threadIdx.x < 3) ? INT_MAX : INT_MIN;
    __syncthreads();
    int x0, y0, z0;
    tile_coords(g, blockIdx.x, x0, y0, z0);
    const int x = x0 + (threadIdx.x % SL_LANES), y = y0 + threadIdx.x / SL_LANES;
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
    if ((int)(threadIdx.x % SL_LANES) < SL_TX && x < g.n1 && y < g.n2) {
        for (int k = 0; k < SL_TZ; ++k) {
            const int z = z0 + k;
            if (z >= g.n3) break;
            const int64_t id = ((int64_t)z * g.n2 + y) * g.n1 + x;
            const int ii[3] = {x, y, z + g.z0};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                T da;
                if constexpr (DSTAR) {
                    da = ds.c[a] * ds.v[a][id];
                    d[a * g.M + id] = da;
                } else {
                    da = d[a * g.M + id];
                }
                int q;
                T t;
                cell_of<T>(ii[a], da, q, t);
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
        if (g.ghost && (p[2] - g.z0 + g.zg < 0 || p[2] + p[5] - g.z0 > g.n3 + g.zgh)) atomicOr(&maxext[3], 1);
    }
}

// ---------------------------------------------------------------------------------------------
// Epilogues of the fused gather kernel.  `late(id)` issues the voxel's pointwise operand loads just
// before its interpolation (they fly while the 64 stencil reads run); `store(id, val, late)` finishes
// the step with the NC interpolated components `val` at the departure point.  Indices are 32-bit
// (M <= 2^30); vector fields are passed as one pointer per component.
struct NoLate {};

template <typename T>
struct EpiStore {  // state solve: rho_{j+1} = I[rho_j](X+)   (Eq. 7 with f = 0)
    T* out;
    using Late = NoLate;
    __device__ __forceinline__ Late late(uint32_t) const { return Late{}; }
    __device__ __forceinline__ T store(uint32_t id, const T* val, const Late&) const {
        out[id] = val[0];
        return val[0];
    }
};

// Adjoint-like step: nu_{k-1} = scale * m * I[nu_k](X-)  (Eq. 7 with f = nu div v; D7).
// QUAD != 0 also accumulates the trapezoid quadrature b~ = dt sum_j w_j lambda~_j G_j (P:L196-198,
// reading A12) step by step, so the streaming sum rides on the gather's shared-memory-bound time:
// QUAD = 1 (first step, k = nt, full Newton): b~ = w_nt nu_nt G_nt + w_{nt-1} nu_{nt-1} G_{nt-1}, nu_nt
// read at x; QUAD = 2: b~ += w_{k-1} nu_{k-1} G_{k-1} (every GN step: the k = nt term was written by the
// last incremental-state step, EpiIncState<T, true>).
// NEWTON (NEXT-3, full-Newton incremental adjoint, Eq. 5c with div(lam vt)): the gather carries a
// second component, I[s_k](X) with s_k = div(lam_k vt) at the old level, and Eq. 7 gives
//   nu_{k-1} = m I[nu_k](X) + dt/2 (1 + dt D(x)) I[s_k](X) + dt/2 s_{k-1}(x)   (D = div v; 0 isochoric).
template <typename T, int QUAD = 0, bool NEWTON = false>
struct EpiAdjoint {
    T* out;        // nu_{k-1}
    const T* m;    // nullable (isochoric: m == 1)
    T scale;
    // quadrature operands (QUAD != 0)
    T* b0; T* b1; T* b2;                     // b~ components (read-modify-write when QUAD == 2)
    const T* G0; const T* G1; const T* G2;   // G_{k-1}
    T w;                                     // dt w_{k-1}
    const T* nu; T snu;                      // QUAD == 1: nu_nt = snu * nu[x]
    const T* H0; const T* H1; const T* H2;   // QUAD == 1: G_nt
    T wn;                                    // QUAD == 1: dt w_nt
    // NEWTON operands
    const T* D;                              // div v at x (nullable: isochoric)
    const T* snew;                           // s_{k-1} at x
    T hdt, dtt;                              // dt / 2, dt
    // late() only loads: arithmetic on a loaded value here would stall the warp on the load right away
    // instead of a pair later (store() does all of it; same operations in the same order)
    struct Late { T m; T g[3]; T b[3]; T Dx, sn, nu; };
    __device__ __forceinline__ Late late(uint32_t id) const {
        Late l;
        l.m = m ? __ldg(m + id) : T(1);
        if constexpr (NEWTON) {
            l.Dx = D ? __ldg(D + id) : T(0);
            l.sn = __ldg(snew + id);
        }
        if constexpr (QUAD != 0) {
            l.g[0] = __ldg(G0 + id);
            l.g[1] = __ldg(G1 + id);
            l.g[2] = __ldg(G2 + id);
            if constexpr (QUAD == 2) {
                l.b[0] = b0[id];
                l.b[1] = b1[id];
                l.b[2] = b2[id];
            } else {  // G_nt (the b~ term of nu_nt) parked in b
                l.nu = __ldg(nu + id);
                l.b[0] = __ldg(H0 + id);
                l.b[1] = __ldg(H1 + id);
                l.b[2] = __ldg(H2 + id);
            }
        }
        return l;
    }
    __device__ __forceinline__ T store(uint32_t id, const T* val, const Late& l) const {
        const T mm = m ? scale * l.m : scale;
        T r = mm * val[0];
        if constexpr (NEWTON) r += hdt * (T(1) + dtt * l.Dx) * val[1] + hdt * l.sn;
        out[id] = r;
        if constexpr (QUAD != 0) {
            T b[3] = {l.b[0], l.b[1], l.b[2]};
            if constexpr (QUAD == 1) {
                const T ln = wn * snu * l.nu;
                b[0] = ln * l.b[0];
                b[1] = ln * l.b[1];
                b[2] = ln * l.b[2];
            }
            const T wr = w * r;
            b0[id] = b[0] + wr * l.g[0];
            b1[id] = b[1] + wr * l.g[1];
            b2[id] = b[2] + wr * l.g[2];
        }
        return r;
    }
};

template <typename T>
struct EpiAddScaled {  // out = I[w](X) + c f(x): the merged-source step of the deformation map (NEXT-4)
    T* out;
    const T* f;
    T c;
    struct Late { T f; };
    __device__ __forceinline__ Late late(uint32_t id) const { return Late{__ldg(f + id)}; }
    __device__ __forceinline__ T store(uint32_t id, const T* val, const Late& l) const {
        const T r = val[0] + c * l.f;
        out[id] = r;
        return r;
    }
};

// WB (last step, j + 1 = nt): also starts the b~ quadrature with its k = nt term
// w_nt lambda~_nt G_nt, lambda~_nt = -rho~_nt: b~ = (wq rho~_nt) G_nt with wq = -w_nt = -dt/2.  G_nt is
// this step's source gradient, already in registers, so the term costs three stores here instead of
// four loads in the first adjoint step.
template <typename T, bool WB = false>
struct EpiIncState {  // Algorithm 2 with the merged gather: g_{j+1} = I[g_j](X+) + c f_{j+1}, f = -vt.G_{j+1}
    T* out;
    const T* vt0; const T* vt1; const T* vt2;  // vt components
    const T* G0; const T* G1; const T* G2;     // grad rho_{j+1} components
    T c;
    T* b0 = nullptr; T* b1 = nullptr; T* b2 = nullptr;  // WB: b~ components
    T wq = T(0);                                        // WB: w_nt * snu
    struct Late { T v[3], g[3]; };
    __device__ __forceinline__ Late late(uint32_t id) const {
        return Late{{__ldg(vt0 + id), __ldg(vt1 + id), __ldg(vt2 + id)}, {__ldg(G0 + id), __ldg(G1 + id), __ldg(G2 + id)}};
    }
    __device__ __forceinline__ T store(uint32_t id, const T* val, const Late& l) const {
        const T f = l.v[0] * l.g[0] + l.v[1] * l.g[1] + l.v[2] * l.g[2];
        const T r = val[0] - c * f;
        out[id] = r;
        if constexpr (WB) {  // same products as EpiAdjoint<T, 1>::store
            const T ln = wq * r;
            b0[id] = ln * l.g[0];
            b1[id] = ln * l.g[1];
            b2[id] = ln * l.g[2];
        }
        return r;
    }
};

template <typename T>
struct EpiMultiplier {  // m = 1 + dt/2 (Dbar + D + dt Dbar D), Dbar = I[div v](X-)  (D7)
    T* m;
    const T* D;
    T dt;
    struct Late { T D; };
    __device__ __forceinline__ Late late(uint32_t id) const { return Late{__ldg(D + id)}; }
    __device__ __forceinline__ T store(uint32_t id, const T* val, const Late& l) const {
        const T Db = val[0];
        const T r = T(1) + T(0.5) * dt * (Db + l.D + dt * Db * l.D);
        m[id] = r;
        return r;
    }
};

template <typename T>
struct EpiDeparture1 {  // d_a = sigma dt/2 (v_a(x) + I[v_a](X*)) / h_a  (Eq. 6, cell units), one component a:
    T* d;               // three one-component gathers (54 KB boxes, 4 CTAs/SM) beat one three-component
                        // gather (173 KB box, 1 CTA/SM): 3 x ? vs 686 us at 256^3
    const T* v;
    T c;
    struct Late { T v; };
    __device__ __forceinline__ Late late(uint32_t id) const { return Late{__ldg(v + id)}; }
    __device__ __forceinline__ T store(uint32_t id, const T* val, const Late& l) const {
        const T r = c * (l.v + val[0]);
        d[id] = r;
        return r;
    }
};

// Fused ghost exchange (multi-GPU x3 slabs): the gather that produces a field which the
// next gather reads also stores the slab's boundary planes straight into the x3 neighbours' ghost planes
// of the same slot (peer memory: NVLink stores to a CUDA-IPC-mapped workspace with one process per GPU,
// the other contexts' workspaces with loopback ranks).  Planes z < zgh go to the lower neighbour's upper
// ghosts, planes z >= n3 - zg to the upper neighbour's lower ghosts; the consumer then only waits for its
// neighbours (Impl::peer_sync) instead of exchanging ghost planes before its gather.
template <typename T, class Epi>
struct EpiPeer {
    Epi e;
    T* lo;              // lo[id] = lower neighbour's upper ghost of my voxel id (id < lo_end)
    T* hi;              // hi[id] = upper neighbour's lower ghost of my voxel id (id >= hi_begin)
    uint32_t lo_end, hi_begin;
    using Late = typename Epi::Late;
    __device__ __forceinline__ Late late(uint32_t id) const { return e.late(id); }
    __device__ __forceinline__ T store(uint32_t id, const T* val, const Late& l) const {
        const T r = e.store(id, val, l);
        if (id < lo_end) lo[id] = r;
        if (id >= hi_begin) hi[id] = r;
        return r;
    }
};

template <typename T, int NC>
struct Src {
    const T* p[NC];
};
template <typename T>
struct Disp {  // displacement field components (cell units)
    const T* p[3];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Shared-memory box geometry per (value type, components): compile-time strides so every one of the
// 64 stencil loads is an LDS with an immediate offset from one per-point base address.  The row and
// plane strides are multiples of 32 words: the 32 lanes of a warp read consecutive columns, so when
// their departure rows or planes differ (the displacement crosses a cell boundary along x) they still
// hit 32 distinct banks.  BX holds a 32-wide tile's x-extent (32 + 3 + deformation spread + 16-B
// alignment), BY/BZ an 8-deep tile's.
template <typename T, int NC>
struct BoxGeom;
// MINB: CTAs per SM the register budget must allow.
template <> struct BoxGeom<float, 1> { static constexpr int BX = 64, BY = 15, BZ = 14, MINB = 4; };   // 54 KB
template <> struct BoxGeom<float, 2> { static constexpr int BX = 64, BY = 15, BZ = 15, MINB = 1; };   // 115 KB
template <> struct BoxGeom<float, 3> { static constexpr int BX = 64, BY = 15, BZ = 15, MINB = 1; };   // 173 KB
template <> struct BoxGeom<double, 1> { static constexpr int BX = 64, BY = 15, BZ = 15, MINB = 1; };  // 115 KB
template <> struct BoxGeom<double, 2> { static constexpr int BX = 48, BY = 14, BZ = 14, MINB = 1; };  // 150 KB
template <> struct BoxGeom<double, 3> { static constexpr int BX = 48, BY = 14, BZ = 14, MINB = 1; };  // 221 KB

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

// Two points at once with packed fp32x2 arithmetic (sm_100 FFMA2): lane .x = point A, .y = point B.
__device__ __forceinline__ void lagrange4x2(float2 t, float2 w[4]) {
    const float2 a = __fmul2_rn(t, __fadd2_rn(t, make_float2(-1.f, -1.f)));   // t (t - 1)
    const float2 b = __fadd2_rn(a, make_float2(-2.f, -2.f));                    // (t + 1)(t - 2)
    const float s = 1.f / 6.f;
    w[0] = __fmul2_rn(a, __ffma2_rn(t, make_float2(-s, -s), make_float2(2.f * s, 2.f * s)));
    w[1] = __fmul2_rn(b, __ffma2_rn(t, make_float2(0.5f, 0.5f), make_float2(-0.5f, -0.5f)));
    w[2] = __fmul2_rn(b, __fmul2_rn(t, make_float2(-0.5f, -0.5f)));
    w[3] = __fmul2_rn(a, __ffma2_rn(t, make_float2(s, s), make_float2(s, s)));
}

template <int BX, int BY>
__device__ __forceinline__ float2 interp_box2(const float* __restrict__ bA, const float* __restrict__ bB,
                                              const float2 w1[4], const float2 w2[4], const float2 w3[4]) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float2 accb = make_float2(0.f, 0.f);
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const float* rA = bA + (c * BY + bb) * BX;
            const float* rB = bB + (c * BY + bb) * BX;
            float2 row = __fmul2_rn(w1[0], make_float2(rA[0], rB[0]));
            row = __ffma2_rn(w1[1], make_float2(rA[1], rB[1]), row);
            row = __ffma2_rn(w1[2], make_float2(rA[2], rB[2]), row);
            row = __ffma2_rn(w1[3], make_float2(rA[3], rB[3]), row);
            accb = (bb == 0) ? __fmul2_rn(w2[0], row) : __ffma2_rn(w2[bb], row, accb);
        }
        acc = (c == 0) ? __fmul2_rn(w3[0], accb) : __ffma2_rn(w3[c], accb, acc);
    }
    return acc;
}

#ifdef DR_TAPROT
// A/B experiment only (tools/bank_sim.py --rotated; never the product build): each lane reads the four
// x1 taps of a stencil row rotated by floor(-d1) mod 4, so lanes whose x1 floors differ by one read
// the same column offset from their own x in 3 of the 4 loads.  Sums in the rotated order.
__device__ __forceinline__ float pick4(const float2 w[4], int i, bool y) {
    const float v0 = y ? w[0].y : w[0].x, v1 = y ? w[1].y : w[1].x, v2 = y ? w[2].y : w[2].x,
                v3 = y ? w[3].y : w[3].x;
    const float lo = (i & 1) ? v1 : v0, hi = (i & 1) ? v3 : v2;
    return (i & 2) ? hi : lo;
}
template <int BX, int BY>
__device__ __forceinline__ float2 interp_box2_rot(const float* const pA[4], const float* const pB[4],
                                                  const float2 w1[4], const float2 w2[4], const float2 w3[4]) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float2 accb = make_float2(0.f, 0.f);
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const int o = (c * BY + bb) * BX;
            float2 row = __fmul2_rn(w1[0], make_float2(pA[0][o], pB[0][o]));
            row = __ffma2_rn(w1[1], make_float2(pA[1][o], pB[1][o]), row);
            row = __ffma2_rn(w1[2], make_float2(pA[2][o], pB[2][o]), row);
            row = __ffma2_rn(w1[3], make_float2(pA[3][o], pB[3][o]), row);
            accb = (bb == 0) ? __fmul2_rn(w2[0], row) : __ffma2_rn(w2[bb], row, accb);
        }
        acc = (c == 0) ? __fmul2_rn(w3[0], accb) : __ffma2_rn(w3[c], accb, acc);
    }
    return acc;
}
#endif

// Tile context: origin of the tile and the planned box (x origin aligned down to VEC = 16 B /
// sizeof(T) so rows stage as 16-byte cp.async chunks; N1 is a multiple of VEC, so a chunk never
// straddles the periodic wrap).
template <typename T, int NC>
struct TileCtx {
    int x0, y0, z0, ox, oy, oz, ex, ey, ez;
    bool fits;
};

// WIN: the box of the sliding-window gather (k_sl_window), one cell wider: +1 on the high side of x1
// and x2 (a thread's 5-wide window starts at its lowest stencil node), +1 on both sides of x3 (its
// 12-plane window may start one plane below the tile's lowest node or end one above the highest).
template <typename T, int NC, class Geo = BoxGeom<T, NC>, bool WIN = false>
__device__ __forceinline__ TileCtx<T, NC> tile_ctx(const Grid& g, const int* __restrict__ plan, int tile) {
    constexpr int VEC = 16 / (int)sizeof(T);
    constexpr int BX = Geo::BX, BY = Geo::BY, BZ = Geo::BZ;
    TileCtx<T, NC> c;
    tile_coords(g, tile, c.x0, c.y0, c.z0);
    const int4 p = __ldg(reinterpret_cast<const int4*>(plan + (size_t)tile * PLAN_INTS));
    const int4 q = __ldg(reinterpret_cast<const int4*>(plan + (size_t)tile * PLAN_INTS + 4));
    c.ox = p.x & ~(VEC - 1);
    c.oy = p.y;
    c.oz = p.z - (WIN ? 1 : 0);
    c.ex = ((p.x + p.w + (WIN ? 1 : 0) - c.ox) + VEC - 1) & ~(VEC - 1);
    c.ey = q.x + (WIN ? 1 : 0);
    c.ez = q.y + (WIN ? 2 : 0);
    c.fits = c.ex <= BX && c.ey <= BY && c.ez <= BZ;
    // slabs: a box leaving the planes + ghosts holds points served by their owner rank (scatter)
    if (g.ghost && (c.oz - g.z0 + g.zg < 0 || c.oz + c.ez - g.z0 > g.n3 + g.zgh)) c.fits = false;
    return c;
}

template <typename T, int NC, class Geo = BoxGeom<T, NC>>
__device__ __forceinline__ void stage_box(const Grid& g, const Src<T, NC>& src, const TileCtx<T, NC>& c, T* box) {
    constexpr int VEC = 16 / (int)sizeof(T);
    constexpr int BX = Geo::BX, BY = Geo::BY, BZ = Geo::BZ;
    constexpr int SC = BX * BY * BZ;
    constexpr int NCHP = BX / VEC;
    constexpr int RSTEP = SL_THREADS / NCHP;
    if (!c.fits) return;
    const int nch = c.ex / VEC;
    const int ch = threadIdx.x % NCHP;
    const int r0 = threadIdx.x / NCHP;
    if (ch >= nch || r0 >= RSTEP) return;
    int yy = r0, zz = 0;
    while (yy >= c.ey) { yy -= c.ey; ++zz; }
    const int gx = wrap2(c.ox + ch * VEC, g.n1);  // N1 % VEC == 0: a chunk never straddles the wrap
    while (zz < c.ez) {
        const int gy = wrap2(c.oy + yy, g.n2);
        const int gz = g.ghost ? c.oz + zz - g.z0 + g.zg : wrap2(c.oz + zz, g.n3);
        const uint32_t gofs = ((uint32_t)gz * g.n2 + gy) * g.n1 + gx;
        T* dst = box + (zz * BY + yy) * BX + ch * VEC;
        DR_ASSERT(zz < BZ && yy < BY && ch * VEC + VEC <= BX && gz >= 0 && gz < g.n3 + g.zg + g.zgh);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) cp_async16(dst + cc * SC, src.p[cc] + gofs);
        yy += RSTEP;
        while (yy >= c.ey) { yy -= c.ey; ++zz; }
    }
}

// Operands of one pair of points (k, k + 4) of a thread: displacements and the epilogue's pointwise
// operands.  They are loaded one pair ahead (pair 0 together with the box staging), so every global
// load has a whole pair's interpolation (~300 instructions per warp) to land.
template <typename T, class Epi>
struct PairIn {
    T dA[3], dB[3];
    typename Epi::Late lA, lB;
};

template <typename T, class Epi>
__device__ __forceinline__ void load_pair(const Disp<T>& d, const Epi& epi, uint32_t idA, uint32_t idB, bool okA,
                                          bool okB, PairIn<T, Epi>& in) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        in.dA[a] = okA ? __ldg(d.p[a] + idA) : T(0);
        in.dB[a] = okB ? __ldg(d.p[a] + idB) : T(0);
    }
    if (okA) in.lA = epi.late(idA);
    if (okB) in.lB = epi.late(idB);
}

// Interpolate a pair from the staged box and finish both points.
template <typename T, int NC, class Epi, class Geo = BoxGeom<T, NC>>
__device__ __forceinline__ void pair_from_box(const Grid& g, const TileCtx<T, NC>& c, const T* __restrict__ box,
                                              int x, int y, int zA, uint32_t idA, uint32_t idB, bool okB,
                                              const PairIn<T, Epi>& in, const Epi& epi) {
    constexpr int BX = Geo::BX, BY = Geo::BY, BZ = Geo::BZ;
    constexpr int SC = BX * BY * BZ;
    constexpr int H = SL_TZ / 2;
    int qA[3], qB[3];
    T tA[3], tB[3];
    const int ii[3] = {x, y, zA + g.z0};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        cell_of<T>(ii[a], in.dA[a], qA[a], tA[a]);
        cell_of<T>(ii[a] + (a == 2 ? H : 0), in.dB[a], qB[a], tB[a]);
        if (!okB) { qB[a] = qA[a]; tB[a] = tA[a]; }
    }
    const T* bA = box + ((qA[2] - 1 - c.oz) * BY + (qA[1] - 1 - c.oy)) * BX + (qA[0] - 1 - c.ox);
    const T* bB = box + ((qB[2] - 1 - c.oz) * BY + (qB[1] - 1 - c.oy)) * BX + (qB[0] - 1 - c.ox);
    DR_ASSERT(qA[0] - 1 - c.ox >= 0 && qA[0] + 2 - c.ox < c.ex && qA[1] - 1 - c.oy >= 0 && qA[1] + 2 - c.oy < c.ey &&
              qA[2] - 1 - c.oz >= 0 && qA[2] + 2 - c.oz < c.ez);
    DR_ASSERT(qB[0] - 1 - c.ox >= 0 && qB[0] + 2 - c.ox < c.ex && qB[1] - 1 - c.oy >= 0 && qB[1] + 2 - c.oy < c.ey &&
              qB[2] - 1 - c.oz >= 0 && qB[2] + 2 - c.oz < c.ez);
    T vA[NC], vB[NC];
    if constexpr (sizeof(T) == 4) {
        float2 w[3][4];
#pragma unroll
        for (int a = 0; a < 3; ++a) lagrange4x2(make_float2(tA[a], tB[a]), w[a]);
#ifdef DR_TAPROT
        const int sA = (qA[0] - x) & 3, sB = (qB[0] - x) & 3;
        const float* pA[4];
        const float* pB[4];
        float2 w1r[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int oA = (a - sA) & 3, oB = (a - sB) & 3;
            pA[a] = bA + oA;
            pB[a] = bB + oB;
            w1r[a] = make_float2(pick4(w[0], oA, false), pick4(w[0], oB, true));
        }
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
            const float* qa[4] = {pA[0] + cc * SC, pA[1] + cc * SC, pA[2] + cc * SC, pA[3] + cc * SC};
            const float* qb[4] = {pB[0] + cc * SC, pB[1] + cc * SC, pB[2] + cc * SC, pB[3] + cc * SC};
            const float2 r = interp_box2_rot<BX, BY>(qa, qb, w1r, w[1], w[2]);
            vA[cc] = r.x;
            vB[cc] = r.y;
        }
#else
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
            const float2 r = interp_box2<BX, BY>(bA + cc * SC, bB + cc * SC, w[0], w[1], w[2]);
            vA[cc] = r.x;
            vB[cc] = r.y;
        }
#endif
    } else {
        T w1[4], w2[4], w3[4];
        lagrange4(tA[0], w1);
        lagrange4(tA[1], w2);
        lagrange4(tA[2], w3);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) vA[cc] = interp_box<T, BX, BY>(bA + cc * SC, w1, w2, w3);
        if (okB) {
            lagrange4(tB[0], w1);
            lagrange4(tB[1], w2);
            lagrange4(tB[2], w3);
#pragma unroll
            for (int cc = 0; cc < NC; ++cc) vB[cc] = interp_box<T, BX, BY>(bB + cc * SC, w1, w2, w3);
        }
    }
    epi.store(idA, vA, in.lA);
    if (okB) epi.store(idB, vB, in.lB);
}

// Fused gather + epilogue.  Grid: one CTA per 32 x 8 x 8 tile; thread = (x, y) column of 8 points,
// processed as 4 pairs (k, k + 4).  Dynamic smem: box_bytes<T, NC>().
// (A) stage the tile's box with 16-byte cp.async (periodic wrap per chunk in x1/x2; x3 wraps, or with
// slabs indexes through the ghost planes); load pair 0's operands meanwhile; (B) wait + barrier;
// (C) per pair: issue the next pair's loads, gather the 64 stencil values per point from shared memory
// -- the two points as one packed fp32x2 pair (FFMA2) -- and finish the step.  Tiles whose box exceeds
// the compile-time capacity gather from global memory instead (same arithmetic, one point at a time).
// Resident CTAs per SM of a gather (fp32, one component): 4 (64 registers) unless the epilogue's
// operands need more registers without spilling (inc-state source, adjoint + quadrature): 3 (80).
template <class Epi>
struct EpiMinB {
    static constexpr int V = 4;
};
#ifndef DR_MINB_INC
#define DR_MINB_INC 3
#endif
#ifndef DR_MINB_Q2
#define DR_MINB_Q2 3
#endif
template <typename T, bool WB>
struct EpiMinB<EpiIncState<T, WB>> {
    static constexpr int V = DR_MINB_INC;
};
template <typename T, bool N>
struct EpiMinB<EpiAdjoint<T, 1, N>> {
    static constexpr int V = 3;
};
template <typename T, bool N>
struct EpiMinB<EpiAdjoint<T, 2, N>> {
    static constexpr int V = DR_MINB_Q2;
};
template <typename T, class Epi>
struct EpiMinB<EpiPeer<T, Epi>> {
    static constexpr int V = EpiMinB<Epi>::V;
};
template <typename T, int NC, class Epi>
struct GatherMinB {
    static constexpr int V = (sizeof(T) == 4 && NC == 1) ? EpiMinB<Epi>::V : BoxGeom<T, NC>::MINB;
};

// Global-memory path of one thread's column of SL_TZ points (tiles whose box exceeds the shared-memory
// capacity; with slabs also the points served by their owner rank are skipped here).
template <typename T, int NC, class Epi>
__device__ __forceinline__ void column_from_global(const Grid& g, const Src<T, NC>& src, const Disp<T>& d, int x,
                                                   int y, int z0, int kmax, uint32_t id0, uint32_t plane,
                                                   const Epi& epi) {
#pragma unroll 1
    for (int k = 0; k < kmax; ++k) {
        const uint32_t id = id0 + k * plane;
        int q1, q2, q3;
        T t1, t2, t3;
        cell_of<T>(x, __ldg(d.p[0] + id), q1, t1);
        cell_of<T>(y, __ldg(d.p[1] + id), q2, t2);
        cell_of<T>(z0 + k + g.z0, __ldg(d.p[2] + id), q3, t3);
        if (g.ghost && (q3 - 1 < g.z0 - g.zg || q3 + 2 >= g.z0 + g.n3 + g.zgh)) continue;  // remote point
        T w1[4], w2[4], w3[4];
        lagrange4(t1, w1);
        lagrange4(t2, w2);
        lagrange4(t3, w3);
        T val[NC];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) val[cc] = interp_global(src.p[cc], g, q1, q2, q3, w1, w2, w3);
        epi.store(id, val, epi.late(id));
    }
}

// Box staging by the tensor-map TMA engine (fp32, one component): a 3-D map over the source's ghosted
// slot (x1, x2, slot planes) with the box's compile-time extents (BoxGeom: 64 x 15 x 14) lands the box
// exactly in the gather's shared-memory layout (row stride 64 words) with one cp.async.bulk.tensor
// issued by one thread and completed on an mbarrier -- no per-chunk address arithmetic or LDGSTS on
// the LSU path the stencil loads saturate.  Only tiles whose planned box does not wrap periodically
// (the map cannot wrap; columns past the field are zero-filled and never read) use it; the others
// stage with cp.async as before.  tm: a zeroed map disables it (use = 0).
struct GatherTma {
    CUtensorMap tm;
    int use;
};
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// the planned box [ox, ox + ex) x [oy, oy + ey) x [oz, oz + ez) lies inside the source slot (no wrap)
template <typename T, int NC>
__device__ __forceinline__ bool box_inside(const Grid& g, const TileCtx<T, NC>& c) {
    const int zs = g.ghost ? c.oz - g.z0 + g.zg : c.oz;
    const int nzs = g.ghost ? g.n3 + g.zg + g.zgh : g.n3;
    return c.fits && c.ox >= 0 && c.ox + c.ex <= g.n1 && c.oy >= 0 && c.oy + c.ey <= g.n2 && zs >= 0 && zs + c.ez <= nzs;
}

template <typename T, int NC, class Epi>
__global__ void __launch_bounds__(SL_THREADS, (GatherMinB<T, NC, Epi>::V))
    k_sl_gather(Grid g, Src<T, NC> src, Disp<T> d, const int* __restrict__ plan, int ntiles, Epi epi) {
    constexpr int H = SL_TZ / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* box = reinterpret_cast<T*>(smem_raw);
    const int tile = blockIdx.x;
    if (tile >= ntiles) return;
    const TileCtx<T, NC> c = tile_ctx<T, NC>(g, plan, tile);
    stage_box<T, NC>(g, src, c, box);
    const int x = c.x0 + (threadIdx.x % SL_LANES), y = c.y0 + threadIdx.x / SL_LANES;
    const bool xyok = (int)(threadIdx.x % SL_LANES) < SL_TX && x < g.n1 && y < g.n2;
    const int kmax = min(SL_TZ, g.n3 - c.z0);
    const uint32_t plane = (uint32_t)g.n1 * (uint32_t)g.n2;
    const uint32_t id0 = ((uint32_t)c.z0 * g.n2 + y) * g.n1 + x;
    if (!c.fits) {  // global-memory fallback (no barrier needed: nothing was staged)
        if (xyok) column_from_global<T, NC, Epi>(g, src, d, x, y, c.z0, kmax, id0, plane, epi);
        return;
    }
    PairIn<T, Epi> cur;
    if (xyok) load_pair<T, Epi>(d, epi, id0, id0 + H * plane, 0 < kmax, H < kmax, cur);
    cp_async_wait_all();
    __syncthreads();
    if (!xyok) return;
#pragma unroll
    for (int p = 0; p < H; ++p) {
        if (p >= kmax) break;
        PairIn<T, Epi> nxt;
        if (p + 1 < H && p + 1 < kmax)
            load_pair<T, Epi>(d, epi, id0 + (p + 1) * plane, id0 + (p + 1 + H) * plane, true, p + 1 + H < kmax, nxt);
        pair_from_box<T, NC, Epi>(g, c, box, x, y, c.z0 + p, id0 + p * plane, id0 + (p + H) * plane, p + H < kmax,
                                  cur, epi);
        cur = nxt;
    }
}

// The same gather with the box staged by the TMA engine where the planned box does not wrap (fp32, one
// component; GatherTma above).
template <class Epi>
__global__ void __launch_bounds__(SL_THREADS, (GatherMinB<float, 1, Epi>::V))
    k_sl_gather_tma(Grid g, Src<float, 1> src, Disp<float> d, const int* __restrict__ plan, int ntiles, Epi epi,
                const __grid_constant__ GatherTma gt) {
    using T = float;
    constexpr int NC = 1;
    constexpr int H = SL_TZ / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t tbar;
    T* box = reinterpret_cast<T*>(smem_raw);
    const int tile = blockIdx.x;
    if (tile >= ntiles) return;
    const TileCtx<T, NC> c = tile_ctx<T, NC>(g, plan, tile);
    bool tma = false;
    {
        tma = box_inside<T, NC>(g, c);  // uniform per CTA
        if (tma) {
            if (threadIdx.x == 0) {
                mbar_init(&tbar, 1);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                mbar_expect(&tbar, (unsigned)box_bytes<T, NC>());
                tma_load_3d(box, &gt.tm, c.ox, c.oy, g.ghost ? c.oz - g.z0 + g.zg : c.oz, &tbar);
            }
        }
    }
    if (!tma) stage_box<T, NC>(g, src, c, box);
    const int x = c.x0 + (threadIdx.x % SL_LANES), y = c.y0 + threadIdx.x / SL_LANES;
    const bool xyok = (int)(threadIdx.x % SL_LANES) < SL_TX && x < g.n1 && y < g.n2;
    const int kmax = min(SL_TZ, g.n3 - c.z0);
    const uint32_t plane = (uint32_t)g.n1 * (uint32_t)g.n2;
    const uint32_t id0 = ((uint32_t)c.z0 * g.n2 + y) * g.n1 + x;
    if (!c.fits) {  // global-memory fallback (no barrier needed: nothing was staged)
        if (xyok) column_from_global<T, NC, Epi>(g, src, d, x, y, c.z0, kmax, id0, plane, epi);
        return;
    }
    PairIn<T, Epi> cur;
    if (xyok) load_pair<T, Epi>(d, epi, id0, id0 + H * plane, 0 < kmax, H < kmax, cur);
    if (tma) {
        __syncthreads();  // the mbarrier's initialisation is visible before anyone waits on it
        mbar_wait(&tbar, 0);
    } else {
        cp_async_wait_all();
        __syncthreads();
    }
    if (!xyok) return;
#pragma unroll
    for (int p = 0; p < H; ++p) {
        if (p >= kmax) break;
        PairIn<T, Epi> nxt;
        if (p + 1 < H && p + 1 < kmax)
            load_pair<T, Epi>(d, epi, id0 + (p + 1) * plane, id0 + (p + 1 + H) * plane, true, p + 1 + H < kmax, nxt);
        pair_from_box<T, NC, Epi>(g, c, box, x, y, c.z0 + p, id0 + p * plane, id0 + (p + H) * plane, p + H < kmax,
                                  cur, epi);
        cur = nxt;
    }
}

// ---------------------------------------------------------------------------------------------
// Sliding-window gather (fp32, one component: every transport step of the hot path).  The gather is
// bound by the shared-memory datapath (64 stencil LDS per point, 1.3 wavefronts each), so this kernel
// loads each staged value once per thread and reuses it for every point that needs it (P:L314
// "Blocking, prefetching, and vectorization").  A thread's SL_TZ points lie on one x3 column; their
// departure cells move with the smooth velocity, so per axis floor(-d) takes at most two adjacent
// values m, m + 1 over the column (checked per warp; otherwise the pair path of k_sl_gather runs on the
// same box).  The thread then reads a window of 5 x1 columns x 5 x2 rows x (SL_TZ + 4) x3 planes: point
// k's 4x4x4 stencil sits at offset e_a = floor(-d_a) - m_a in {0, 1} of each 5-wide axis and at planes
// k + e_3 .. k + e_3 + 3.  Each point's Lagrange weights are padded with one zero per axis (a 5-vector,
// 6 slots in x3 for a pair), so the window is walked with compile-time offsets and no per-lane
// branches: 25 LDS per plane, 300 per 8 points (37.5 per point instead of 64).  Points k, k + 1 are
// packed in fp32x2 (FFMA2 with the shared window value as a broadcast operand).  The products of the
// zero weights are exact zeros, and the non-zero terms are summed in the same order as the pair path,
// so both paths give the same bits (up to the sign of an exact zero).
struct WinGeom {
    static constexpr int BX = 64, BY = 16, BZ = 16;  // 64 KB
};
constexpr size_t win_box_bytes() { return (size_t)WinGeom::BX * WinGeom::BY * WinGeom::BZ * sizeof(float); }
#ifndef DR_WIN_MINB
#define DR_WIN_MINB 2
#endif
#ifndef DR_WIN_LATE
#define DR_WIN_LATE 1
#endif
constexpr int WIN_MINB = DR_WIN_MINB;  // resident CTAs per SM the register budget must allow
constexpr int WIN_LATE = DR_WIN_LATE;  // planes between a pair's epilogue loads and its store

// slot s of a zero-padded weight vector whose 4 Lagrange weights start at slot e + O (e in {0, 1})
template <int S, int O>
__device__ __forceinline__ float pad_slot(const float w0, const float w1, const float w2, const float w3, bool e) {
    constexpr int i0 = S - O, i1 = S - O - 1;  // weight index at e = 0 / e = 1
    const float a = i0 == 0 ? w0 : i0 == 1 ? w1 : i0 == 2 ? w2 : i0 == 3 ? w3 : 0.f;
    const float b = i1 == 0 ? w0 : i1 == 1 ? w1 : i1 == 2 ? w2 : i1 == 3 ? w3 : 0.f;
    return e ? b : a;
}
// pair weight vector (point A at offset eA, point B at offset OB + eB)
template <int NS, int OB>
__device__ __forceinline__ void pad_pair(const float2 w[4], bool eA, bool eB, float2 W[NS]) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        // (s is a compile-time constant after unrolling)
        float a, b;
        switch (s) {
#define DR_PAD_CASE(S)                                                                 \
    case S:                                                                            \
        a = pad_slot<S, 0>(w[0].x, w[1].x, w[2].x, w[3].x, eA);                        \
        b = pad_slot<S, OB>(w[0].y, w[1].y, w[2].y, w[3].y, eB);                       \
        break;
            DR_PAD_CASE(0) DR_PAD_CASE(1) DR_PAD_CASE(2) DR_PAD_CASE(3) DR_PAD_CASE(4) DR_PAD_CASE(5)
#undef DR_PAD_CASE
            default: a = b = 0.f;
        }
        W[s] = make_float2(a, b);
    }
}

template <class Epi>
__global__ void __launch_bounds__(SL_THREADS, WIN_MINB)
    k_sl_window(Grid g, Src<float, 1> src, Disp<float> d, const int* __restrict__ plan, int ntiles, Epi epi) {
    using T = float;
    constexpr int BX = WinGeom::BX, BY = WinGeom::BY;
    constexpr int H = SL_TZ / 2, NP = SL_TZ / 2, NJ = SL_TZ + 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* box = reinterpret_cast<T*>(smem_raw);
    const int tile = blockIdx.x;
    if (tile >= ntiles) return;
    const TileCtx<T, 1> c = tile_ctx<T, 1, WinGeom, true>(g, plan, tile);
    stage_box<T, 1, WinGeom>(g, src, c, box);
    const int x = c.x0 + (threadIdx.x % SL_LANES), y = c.y0 + threadIdx.x / SL_LANES;
    const bool xyok = (int)(threadIdx.x % SL_LANES) < SL_TX && x < g.n1 && y < g.n2;
    const int kmax = min(SL_TZ, g.n3 - c.z0);
    const uint32_t plane = (uint32_t)g.n1 * (uint32_t)g.n2;
    const uint32_t id0 = ((uint32_t)c.z0 * g.n2 + y) * g.n1 + x;
    if (!c.fits) {
        if (xyok) column_from_global<T, 1, Epi>(g, src, d, x, y, c.z0, kmax, id0, plane, epi);
        return;
    }
    // the column's displacements (idle lanes of a narrow grid read a valid column and store nothing)
    const int xc = min((int)(threadIdx.x % SL_LANES) < SL_TX ? x : c.x0, g.n1 - 1), yc = min(y, g.n2 - 1);
    const uint32_t idc = ((uint32_t)c.z0 * g.n2 + yc) * g.n1 + xc;
    bool ok = kmax == SL_TZ;
    float t[3][SL_TZ];
    int fl[3][SL_TZ];
#pragma unroll
    for (int k = 0; k < SL_TZ; ++k)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const T e = ok ? -__ldg(d.p[a] + idc + k * plane) : T(0);
            const T f = floorf(e);
            t[a][k] = e - f;
            fl[a][k] = (int)f;
        }
    int mn[3];
    uint32_t ebits = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int lo = fl[a][0], hi = fl[a][0];
#pragma unroll
        for (int k = 1; k < SL_TZ; ++k) {
            lo = min(lo, fl[a][k]);
            hi = max(hi, fl[a][k]);
        }
        ok = ok && hi - lo <= 1;
        mn[a] = lo;
#pragma unroll
        for (int k = 0; k < SL_TZ; ++k) ebits |= (uint32_t)(fl[a][k] - lo) << (a * SL_TZ + k);
    }
    cp_async_wait_all();
    __syncthreads();
    if (!__all_sync(0xffffffffu, ok)) {  // a deformation too strong for the window: the pair path
        if (!xyok) return;
#pragma unroll 1
        for (int p = 0; p < H; ++p) {
            if (p >= kmax) break;
            PairIn<T, Epi> in;
            load_pair<T, Epi>(d, epi, id0 + p * plane, id0 + (p + H) * plane, true, p + H < kmax, in);
            pair_from_box<T, 1, Epi, WinGeom>(g, c, box, x, y, c.z0 + p, id0 + p * plane, id0 + (p + H) * plane,
                                              p + H < kmax, in, epi);
        }
        return;
    }
    const int col0 = xc + mn[0] - 1 - c.ox, row0 = yc + mn[1] - 1 - c.oy, pl0 = c.z0 + g.z0 + mn[2] - 1 - c.oz;
    DR_ASSERT(col0 >= 0 && col0 + 5 <= c.ex && row0 >= 0 && row0 + 5 <= c.ey && pl0 >= 0 && pl0 + NJ <= c.ez);
    const T* __restrict__ wb = box + (pl0 * BY + row0) * BX + col0;
    float2 W1[NP][5], W2[NP][5], w3[NP][4], acc[NP];  // x3 weights padded per plane (pad_slot)
    bool e3[NP][2];
    typename Epi::Late lt[NP][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        if ((j & 1) == 0 && j / 2 < NP) {  // pair p = (2p, 2p + 1) enters the window at plane 2p
            const int p = j / 2, kA = 2 * p, kB = 2 * p + 1;
            float2 w[4];
            lagrange4x2(make_float2(t[0][kA], t[0][kB]), w);
            pad_pair<5, 0>(w, (ebits >> kA) & 1, (ebits >> kB) & 1, W1[p]);
            lagrange4x2(make_float2(t[1][kA], t[1][kB]), w);
            pad_pair<5, 0>(w, (ebits >> (SL_TZ + kA)) & 1, (ebits >> (SL_TZ + kB)) & 1, W2[p]);
            lagrange4x2(make_float2(t[2][kA], t[2][kB]), w3[p]);
            e3[p][0] = (ebits >> (2 * SL_TZ + kA)) & 1;
            e3[p][1] = (ebits >> (2 * SL_TZ + kB)) & 1;
        }
        if (j >= 5 - WIN_LATE && ((j - 5 + WIN_LATE) & 1) == 0 && (j - 5 + WIN_LATE) / 2 < NP && xyok) {
            const int p = (j - 5 + WIN_LATE) / 2;  // epilogue operands, WIN_LATE planes ahead of the store
            lt[p][0] = epi.late(id0 + 2 * p * plane);
            lt[p][1] = epi.late(id0 + (2 * p + 1) * plane);
        }
        float2 ys[NP];
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            float r[5];
#pragma unroll
            for (int a = 0; a < 5; ++a) r[a] = wb[(j * BY + b) * BX + a];
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (j < 2 * p || j > 2 * p + 5) continue;
                float2 row = __fmul2_rn(W1[p][0], make_float2(r[0], r[0]));
#pragma unroll
                for (int a = 1; a < 5; ++a) row = __ffma2_rn(W1[p][a], make_float2(r[a], r[a]), row);
                ys[p] = b == 0 ? __fmul2_rn(W2[p][0], row) : __ffma2_rn(W2[p][b], row, ys[p]);
            }
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            if (j < 2 * p || j > 2 * p + 5) continue;
            float2 W3;  // slot j - 2p of the pair's 6-slot x3 vector: A at offset e3A, B at 1 + e3B
            switch (j - 2 * p) {
#define DR_W3_CASE(S)                                                                         \
    case S:                                                                                   \
        W3 = make_float2(pad_slot<S, 0>(w3[p][0].x, w3[p][1].x, w3[p][2].x, w3[p][3].x, e3[p][0]),  \
                         pad_slot<S, 1>(w3[p][0].y, w3[p][1].y, w3[p][2].y, w3[p][3].y, e3[p][1])); \
        break;
                DR_W3_CASE(0) DR_W3_CASE(1) DR_W3_CASE(2) DR_W3_CASE(3) DR_W3_CASE(4) DR_W3_CASE(5)
#undef DR_W3_CASE
                default: W3 = make_float2(0.f, 0.f);
            }
            acc[p] = j == 2 * p ? __fmul2_rn(W3, ys[p]) : __ffma2_rn(W3, ys[p], acc[p]);
        }
        if (j >= 5 && ((j - 5) & 1) == 0 && xyok) {  // pair p leaves the window after plane 2p + 5
            const int p = (j - 5) / 2;
            const T vA = acc[p].x, vB = acc[p].y;
            epi.store(id0 + 2 * p * plane, &vA, lt[p][0]);
            epi.store(id0 + (2 * p + 1) * plane, &vB, lt[p][1]);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Shared-plane pair gather (fp32, one component: every transport step of the hot path).  The pair path
// of k_sl_gather is bound by the shared-memory datapath (64 stencil LDS per point at 1.3 wavefronts),
// so this kernel reuses loaded values in registers ("Blocking, prefetching, and vectorization
// can be used to improve the performance").  A thread pairs x3-adjacent points A = (x, y, z) and
// B = (x, y, z + 1).  The velocity is smooth, so on the bench field 93 % of such pairs have equal
// floor(-d) along all three axes (floors differ by a cell along any one axis in 3.3 % of pairs).
// Their stencils then share the same 4 x 4 columns and B's four planes start one plane above A's
// (the box holds that fifth plane: it is B's top stencil plane), so the pair reads the
// 5 planes of the union once (80 LDS for two points instead of 128) and contracts each value with both
// points' weights in one packed FFMA2 (the shared value broadcast).  x3 weights are padded to 5 slots
// (A at slots 0-3, B at 1-4, zeros elsewhere): the zero products are exact zeros, and every
// non-zero term is summed in the pair path's order, so both kernels give the same bits (up to the sign
// of an exact zero).  Pairs that do not share (and the last point of an odd column) are deferred to a
// shared-memory queue that the whole CTA drains after the main loop with the two-pointer pair
// arithmetic (interp_box2), so a misaligned lane idles for one pair instead of making its warp run
// both paths.  Deferred pairs are appended in source-lane order (a misalignment is a smooth surface,
// so neighbouring lanes defer together) and a drain lane takes one pair: neighbouring drain lanes then
// read neighbouring columns, as in the main loop, instead of colliding on random banks.
constexpr int PQ_CAP = SL_THREADS * SL_TZ / 2;  // every pair of the tile (uint16 p * SL_THREADS + thread)
constexpr size_t pairs_smem_bytes() { return box_bytes<float, 1>() + PQ_CAP * sizeof(uint16_t); }

// finish two arbitrary points of the box (either may be invalid: ok = false) with the pair arithmetic
template <class Epi>
__device__ __forceinline__ void pair_any(const Grid& g, const TileCtx<float, 1>& c, const float* __restrict__ box,
                                         const int iA[3], const int iB[3], uint32_t idA, uint32_t idB, bool okA,
                                         bool okB, const float dA[3], const float dB[3],
                                         const typename Epi::Late& lA, const typename Epi::Late& lB, const Epi& epi) {
    constexpr int BX = BoxGeom<float, 1>::BX, BY = BoxGeom<float, 1>::BY;
    int qA[3], qB[3];
    float tA[3], tB[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        cell_of<float>(iA[a], dA[a], qA[a], tA[a]);
        cell_of<float>(iB[a], dB[a], qB[a], tB[a]);
        if (!okB) { qB[a] = qA[a]; tB[a] = tA[a]; }
        if (!okA) { qA[a] = qB[a]; tA[a] = tB[a]; }
    }
    const float* bA = box + ((qA[2] - 1 - c.oz) * BY + (qA[1] - 1 - c.oy)) * BX + (qA[0] - 1 - c.ox);
    const float* bB = box + ((qB[2] - 1 - c.oz) * BY + (qB[1] - 1 - c.oy)) * BX + (qB[0] - 1 - c.ox);
    DR_ASSERT(qA[0] - 1 - c.ox >= 0 && qA[0] + 2 - c.ox < c.ex && qA[1] - 1 - c.oy >= 0 && qA[1] + 2 - c.oy < c.ey &&
              qA[2] - 1 - c.oz >= 0 && qA[2] + 2 - c.oz < c.ez);
    DR_ASSERT(qB[0] - 1 - c.ox >= 0 && qB[0] + 2 - c.ox < c.ex && qB[1] - 1 - c.oy >= 0 && qB[1] + 2 - c.oy < c.ey &&
              qB[2] - 1 - c.oz >= 0 && qB[2] + 2 - c.oz < c.ez);
    float2 w[3][4];
#pragma unroll
    for (int a = 0; a < 3; ++a) lagrange4x2(make_float2(tA[a], tB[a]), w[a]);
    const float2 r = interp_box2<BX, BY>(bA, bB, w[0], w[1], w[2]);
    if (okA) epi.store(idA, &r.x, lA);
    if (okB) epi.store(idB, &r.y, lB);
}

template <class Epi>
__global__ void __launch_bounds__(SL_THREADS, (EpiMinB<Epi>::V))
    k_sl_pairs(Grid g, Src<float, 1> src, Disp<float> d, const int* __restrict__ plan, int ntiles, Epi epi) {
    using T = float;
    constexpr int BX = BoxGeom<T, 1>::BX, BY = BoxGeom<T, 1>::BY;
    constexpr int NP = SL_TZ / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* box = reinterpret_cast<T*>(smem_raw);
    uint16_t* queue = reinterpret_cast<uint16_t*>(smem_raw + box_bytes<T, 1>());
    __shared__ int qn;
    const int tile = blockIdx.x;
    if (tile >= ntiles) return;
    const TileCtx<T, 1> c = tile_ctx<T, 1>(g, plan, tile);
    stage_box<T, 1>(g, src, c, box);
    const int x = c.x0 + (threadIdx.x % SL_LANES), y = c.y0 + threadIdx.x / SL_LANES;
    const bool xyok = (int)(threadIdx.x % SL_LANES) < SL_TX && x < g.n1 && y < g.n2;
    const int kmax = min(SL_TZ, g.n3 - c.z0);
    const uint32_t plane = (uint32_t)g.n1 * (uint32_t)g.n2;
    const uint32_t id0 = ((uint32_t)c.z0 * g.n2 + y) * g.n1 + x;
    if (!c.fits) {  // global-memory fallback (uniform per tile; nothing staged, no barrier)
        if (xyok) column_from_global<T, 1, Epi>(g, src, d, x, y, c.z0, kmax, id0, plane, epi);
        return;
    }
    if (threadIdx.x == 0) qn = 0;
    PairIn<T, Epi> cur;
    if (xyok) load_pair<T, Epi>(d, epi, id0, id0 + plane, 0 < kmax, 1 < kmax, cur);
    cp_async_wait_all();
    __syncthreads();
    if (xyok) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int kA = 2 * p;
            if (kA >= kmax) break;
            const bool okB = kA + 1 < kmax;
            PairIn<T, Epi> nxt;
            if (p + 1 < NP && kA + 2 < kmax)
                load_pair<T, Epi>(d, epi, id0 + (kA + 2) * plane, id0 + (kA + 3) * plane, true, kA + 3 < kmax, nxt);
            const uint32_t idA = id0 + kA * plane, idB = idA + plane;
            const int zA = c.z0 + kA + g.z0;
            int qA[3], qB[3];
            T tA[3], tB[3];
            const int iA[3] = {x, y, zA}, iB[3] = {x, y, zA + 1};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                cell_of<T>(iA[a], cur.dA[a], qA[a], tA[a]);
                cell_of<T>(iB[a], cur.dB[a], qB[a], tB[a]);
            }
            if (okB && qA[0] == qB[0] && qA[1] == qB[1] && qB[2] == qA[2] + 1) {
                const T* bA = box + ((qA[2] - 1 - c.oz) * BY + (qA[1] - 1 - c.oy)) * BX + (qA[0] - 1 - c.ox);
                DR_ASSERT(qA[0] - 1 - c.ox >= 0 && qA[0] + 2 - c.ox < c.ex && qA[1] - 1 - c.oy >= 0 &&
                          qA[1] + 2 - c.oy < c.ey && qA[2] - 1 - c.oz >= 0 && qA[2] + 3 - c.oz < c.ez);
                float2 w1[4], w2[4], w3[4];
                lagrange4x2(make_float2(tA[0], tB[0]), w1);
                lagrange4x2(make_float2(tA[1], tB[1]), w2);
                lagrange4x2(make_float2(tA[2], tB[2]), w3);
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    float2 accb = make_float2(0.f, 0.f);
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        const T* r = bA + (j * BY + bb) * BX;
                        const T r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3];
                        float2 row = __fmul2_rn(w1[0], make_float2(r0, r0));
                        row = __ffma2_rn(w1[1], make_float2(r1, r1), row);
                        row = __ffma2_rn(w1[2], make_float2(r2, r2), row);
                        row = __ffma2_rn(w1[3], make_float2(r3, r3), row);
                        accb = (bb == 0) ? __fmul2_rn(w2[0], row) : __ffma2_rn(w2[bb], row, accb);
                    }
                    // plane j: A's weight j (j < 4), B's weight j - 1 (j > 0)
                    const float2 W = make_float2(j < 4 ? w3[j & 3].x : 0.f, j > 0 ? w3[(j + 3) & 3].y : 0.f);
                    acc = (j == 0) ? __fmul2_rn(W, accb) : __ffma2_rn(W, accb, acc);
                }
                epi.store(idA, &acc.x, cur.lA);
                epi.store(idB, &acc.y, cur.lB);
            } else {  // deferred: slot in source-lane order (warp-aggregated), so drain lanes stay x-adjacent
                const unsigned m = __activemask();
                const unsigned lt = m & ((1u << (threadIdx.x & 31)) - 1u);
                int base = 0;
                if (lt == 0) base = atomicAdd(&qn, __popc(m));
                base = __shfl_sync(m, base, __ffs(m) - 1);
                queue[base + __popc(lt)] = (uint16_t)(p * SL_THREADS + threadIdx.x);
            }
            cur = nxt;
        }
    }
    __syncthreads();
    // drain: one deferred pair per thread (a pair's two points share the thread's column)
    const int n = qn;
    for (int i = threadIdx.x; i < n; i += SL_THREADS) {
        const int e = queue[i];
        const int kA = 2 * (e / SL_THREADS), ts = e % SL_THREADS;
        const bool okB = kA + 1 < kmax;
        const int xs = c.x0 + ts % SL_LANES, ys = c.y0 + ts / SL_LANES;
        const int iA[3] = {xs, ys, c.z0 + kA + g.z0}, iB[3] = {xs, ys, c.z0 + kA + 1 + g.z0};
        const uint32_t idA = ((uint32_t)(c.z0 + kA) * g.n2 + ys) * g.n1 + xs, idB = idA + plane;
        PairIn<T, Epi> in;
        load_pair<T, Epi>(d, epi, idA, idB, true, okB, in);
        pair_any<Epi>(g, c, box, iA, iB, idA, idB, true, okB, in.dA, in.dB, in.lA, in.lB, epi);
    }
}

// ---------------------------------------------------------------------------------------------
// Off-rank departure points (slabs; the paper's Algorithm 1, on x3 slabs).  A point whose
// stencil planes floor(s3)-1 .. floor(s3)+2 leave the rank's planes + ghosts is served by the rank
// owning plane floor(s3): its cell (q, t) travels there once per velocity (the plan), and every gather
// the owner interpolates the requested values and returns them; the requester finishes the step with
// the same epilogue (k_remote_fixup).  Interpolation uses interp_global on both sides of the ghosts,
// so results are the single-rank arithmetic.
template <typename T>
struct RemoteRec {
    int q[3];
    T t[3];
};

__device__ __forceinline__ int remote_owner(const Grid& g, int q3) {
    int w = q3 % g.n3g;
    if (w < 0) w += g.n3g;
    return w / g.n3;
}

// pass 0: count remote points per owner rank; pass 1: write ids and records (slot = off + cursor)
template <typename T>
__global__ void k_remote_classify(Grid g, Disp<T> d, int pass, int* __restrict__ cnt, const int* __restrict__ off,
                                  int* __restrict__ cursor, int* __restrict__ ids, RemoteRec<T>* __restrict__ rec,
                                  int cap) {
    const uint32_t plane = (uint32_t)g.n1 * (uint32_t)g.n2;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.M; e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e % g.n1), y = (int)((e / g.n1) % g.n2), z = (int)(e / plane);
        int q3;
        T t3;
        cell_of<T>(z + g.z0, __ldg(d.p[2] + e), q3, t3);
        if (!(q3 - 1 < g.z0 - g.zg || q3 + 2 >= g.z0 + g.n3 + g.zgh)) continue;
        const int dst = remote_owner(g, q3);
        if (pass == 0) {
            atomicAdd(&cnt[dst], 1);
            continue;
        }
        const int slot = off[dst] + atomicAdd(&cursor[dst], 1);
        if (slot >= cap) continue;  // capacity is checked on the host before this pass
        int q1, q2;
        T t1, t2;
        cell_of<T>(x, __ldg(d.p[0] + e), q1, t1);
        cell_of<T>(y, __ldg(d.p[1] + e), q2, t2);
        ids[slot] = (int)e;
        RemoteRec<T> r;
        r.q[0] = q1;
        r.q[1] = q2;
        int w = q3 % g.n3g;
        r.q[2] = w < 0 ? w + g.n3g : w;
        r.t[0] = t1;
        r.t[1] = t2;
        r.t[2] = t3;
        rec[slot] = r;
    }
}

// owner side: interpolate NC ghosted source fields at n incoming cells
template <typename T, int NC>
__global__ void k_remote_eval(Grid g, Src<T, NC> src, const RemoteRec<T>* __restrict__ rec, int n, T* __restrict__ val) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const RemoteRec<T> r = rec[i];
        T w1[4], w2[4], w3[4];
        lagrange4(r.t[0], w1);
        lagrange4(r.t[1], w2);
        lagrange4(r.t[2], w3);
#pragma unroll
        for (int c = 0; c < NC; ++c) val[(size_t)i * NC + c] = interp_global(src.p[c], g, r.q[0], r.q[1], r.q[2], w1, w2, w3);
    }
}

// requester side: finish the step for its remote points with the returned values
template <typename T, int NC, class Epi>
__global__ void k_remote_fixup(const int* __restrict__ ids, const T* __restrict__ val, int n, Epi epi) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t id = (uint32_t)ids[i];
        T v[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = val[(size_t)i * NC + c];
        epi.store(id, v, epi.late(id));
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
