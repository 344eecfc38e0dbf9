// plane2d.cuh -- fused x1/x2 plane transforms through a thread-block cluster's distributed shared memory
// (one rank, N1 = N2 = 256).  The spectral operators (§III-C1: "N2 N3 1D FFTs across the first
// coordinate ... followed by ... across the second") run per axis as separate HBM passes in fft.cuh;
// here the x1 and x2 transforms of one x3 plane are done in one kernel, so the x1 half spectrum never
// goes to HBM (it was a full write + read of the widest intermediate: complex128 in the forward
// direction).  Per plane, a cluster of CL = 8 CTAs (one per SM):
//   forward  (phase A) CTA r transforms rows i2 = 32r .. 32r + 31 along x1 (r2c) into its shared memory;
//            cluster barrier; (phase B) CTA r transforms the 16 half-spectrum columns k1 = 16r .. 16r + 15
//            along x2, reading the 256 rows of each column from the 8 CTAs' shared memory (DSMEM), and
//            writes the 2-D spectrum to HBM;
//   inverse  (phase B) CTA r inverse-transforms its 16 columns along x2 reading HBM and stores each row
//            of the result into the shared memory of the CTA owning that row (DSMEM); cluster barrier;
//            (phase A) c2r along x1 of its 32 rows, + the epilogue operand, to HBM.
// The 129 half-spectrum columns map onto 8 x 16 = 128 complex column transforms: the k1 = 0 and
// k1 = N1/2 columns are real sequences along x2 after the x1 r2c (X_0 = sum x, X_{N/2} = alternating
// sum), so column slot 0 carries Z = X_0 + i X_{N/2}; forward, the x2 spectrum separates them as
// X_0[k] = (Z_k + conj Z_{-k}) / 2, X_{N/2}[k] = (Z_k - conj Z_{-k}) / 2i (the standard two-real-in-one
// DFT); inverse, Z = X_0 + i X_{N/2} inverse-transforms to (x_0, x_{N/2}) in its real / imaginary part.
// Two shared-memory row buffers alternate between planes, so one cluster barrier per plane orders
// every remote access (the buffer a plane's phase A writes was last read remotely before the previous
// plane's barrier); the other buffer is the column exchange buffer of the plane's phase B.
// The forward input rows of the next plane are fetched by the bulk-copy engine during the current one.
#pragma once
#include "fft.cuh"

namespace dr {

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_id() {
    unsigned r;
    asm("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_count() {
    unsigned r;
    asm("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// generic address of the same shared-memory object in CTA `rank` of the cluster
template <typename T>
__device__ __forceinline__ T* peer_smem(T* p, unsigned rank) {
    uint64_t out;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"((uint64_t)p), "r"(rank));
    return reinterpret_cast<T*>(out);
}

template <typename Tc>
struct Plane2DCfg {
    static constexpr int N = 256, L1 = N / 2, CL = 8, RPC = N / CL, CPC = L1 / CL, NT = 256;
    static constexpr int TPLA = Tpl<L1, Tc>::V;  // row phase: threads per x1 line (8)
    static constexpr int TPLB = Tpl<N, Tc>::V;   // column phase: threads per x2 line (16)
    static_assert(RPC * TPLA == NT && CPC * TPLB == NT, "256 threads per phase");
    static constexpr int LPA = RowLP<L1, Tc, TPLA>::V;
    static constexpr int LPB = ColLP<N, Tc, CPC>::V;
    static constexpr size_t ES = sizeof(Cx<Tc>);
    static constexpr size_t BUFB = (((size_t)(RPC * LPA > CPC * LPB ? RPC * LPA : CPC * LPB) * ES) + 127) & ~(size_t)127;
};

// column element p (row i2 = p) of column x of the x1 half spectra held by the cluster's CTAs
template <typename Tc>
struct PeerColLd {
    Cx<Tc>* rows;  // this CTA's row buffer (same offset in every CTA)
    int x;
    __device__ __forceinline__ Cx<Tc> ld(int p) const {
        using C = Plane2DCfg<Tc>;
        return *peer_smem(rows + (p % C::RPC) * C::LPA + P(x), (unsigned)(p / C::RPC));
    }
};
template <typename Tc>
struct PeerColSt {
    Cx<Tc>* rows;
    int x;
    __device__ __forceinline__ void st(int p, const Cx<Tc>& v) const {
        using C = Plane2DCfg<Tc>;
        *peer_smem(rows + (p % C::RPC) * C::LPA + P(x), (unsigned)(p / C::RPC)) = v;
    }
};
// forward phase B output: the 2-D spectrum row p, column x (slot 0 parks Z in shared memory)
template <typename Tc>
struct SpecColSt {
    Cx<Tc>* g;  // spectrum + (z N) n1p + x
    int rs;     // n1p
    Cx<Tc>* zc;
    __device__ __forceinline__ void st(int p, const Cx<Tc>& v) const {
        if (zc) zc[p] = v;
        else g[(int64_t)p * rs] = v;
    }
};
// inverse phase B input: spectrum column x; slot 0 packs Z = X_0 + i X_{N/2}
template <typename T>
struct SpecColLd {
    const Cx<T>* g;
    int rs;
    int nyq;  // offset of column N/2 from column 0 (slot 0 only), else 0
    __device__ __forceinline__ Cx<T> ld(int p) const {
        const Cx<T> a = g[(int64_t)p * rs];
        if (!nyq) return a;
        const Cx<T> b = g[(int64_t)p * rs + nyq];
        return cx(a.re - b.im, a.im + b.re);
    }
};

// Forward: real planes (Ti) -> 2-D half spectra (Tc), spectrum row stride n1p; nitems = ncomp * n3
// planes, item = comp * n3 + z.  Grid: clusters of CL CTAs, persistent over items.
template <typename Ti, typename Tc>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256, 1)
    k_plane_fwd(const Ti* __restrict__ f, Cx<Tc>* __restrict__ spec, int n3, int nitems, int64_t csf, int64_t css,
                int n1p, const Cx<Tc>* __restrict__ twx, const Cx<Tc>* __restrict__ twy) {
    using C = Plane2DCfg<Tc>;
    constexpr int N = C::N, L1 = C::L1, RPC = C::RPC, CPC = C::CPC;
    constexpr int SI = staged_stride<Ti, C::TPLA>(L1) * (int)sizeof(Cx<Ti>);  // staged input row, bytes
    constexpr size_t STG = (size_t)RPC * SI;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* stg = smem_raw + 128;
    Cx<Tc>* buf0 = reinterpret_cast<Cx<Tc>*>(stg + 2 * STG);
    Cx<Tc>* zc = reinterpret_cast<Cx<Tc>*>(reinterpret_cast<unsigned char*>(buf0) + 2 * C::BUFB);
    const unsigned r = cluster_rank(), cid = cluster_id(), ncl = cluster_count();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int item, int st) {  // rows 32r .. 32r + 31 of the item's plane (contiguous)
        const int comp = item / n3, z = item % n3;
        const unsigned char* src = reinterpret_cast<const unsigned char*>(f + comp * csf + ((int64_t)z * N + r * RPC) * N);
        issue_rows(stg + st * STG, src, 0, RPC, (int64_t)N * sizeof(Ti), SI, N * sizeof(Ti), &bar[st], lane);
    };
    if (warp == 0 && (int)cid < nitems) issue((int)cid, 0);
    const int la = threadIdx.x / C::TPLA, ta = threadIdx.x % C::TPLA;  // row phase: line, thread in line
    const int xb = threadIdx.x % CPC, tb = threadIdx.x / CPC;         // column phase
    int it = 0;
    for (int item = (int)cid; item < nitems; item += (int)ncl, ++it) {
        const int st = it & 1;
        Cx<Tc>* rows = buf0 + (size_t)st * (C::BUFB / C::ES);
        Cx<Tc>* xch = buf0 + (size_t)(st ^ 1) * (C::BUFB / C::ES);
        if (warp == 0 && item + (int)ncl < nitems) issue(item + (int)ncl, st ^ 1);
        mbar_wait(&bar[st], (unsigned)(it >> 1) & 1u);
        // phase A: x1 r2c of row 32r + la (z_n = x_2n + i x_2n+1, L1-point FFT, pair post-processing)
        Cx<Tc>* ln = rows + la * C::LPA;
        const Cx<Ti>* in = reinterpret_cast<const Cx<Ti>*>(stg + st * STG + la * SI);
        fft_line_io<Tc, L1, -1, false, true>(ln, ta, twx, 2, RowLd<Ti, Tc>{in}, SmemLine<Tc>{ln});
        for (int k = ta; k <= L1 / 2; k += C::TPLA) {
            Cx<Tc> Xk, Xl;
            r2c_pair(ln[P(k)], ln[P(k == 0 ? 0 : L1 - k)], twx[k], Xk, Xl);
            if (k == 0) ln[P(0)] = cx(Xk.re, Xl.re);  // X_0 and X_{N1/2}: real
            else {
                ln[P(k)] = Xk;
                if (2 * k != L1) ln[P(L1 - k)] = Xl;
            }
        }
        cluster_sync_all();
        // phase B: x2 FFT of column slot x = 16r + xb (rows from every CTA of the cluster)
        const int comp = item / n3, z = item % n3;
        const int x = (int)r * CPC + xb;
        Cx<Tc>* out = spec + comp * css + (int64_t)z * N * n1p;
        fft_line_io<Tc, N, -1, false, false>(xch + xb * C::LPB, tb, twy, 1, PeerColLd<Tc>{rows, x},
                                             SpecColSt<Tc>{out + x, n1p, x == 0 ? zc : nullptr});
        if (r == 0) {  // separate X_0 and X_{N1/2} from the slot-0 column Z
            __syncthreads();
            const int p = threadIdx.x;
            const Cx<Tc> a = zc[p], b = conj(zc[(N - p) & (N - 1)]);
            out[(int64_t)p * n1p] = cx((a.re + b.re) * Tc(0.5), (a.im + b.im) * Tc(0.5));
            out[(int64_t)p * n1p + L1] = cx((a.im - b.im) * Tc(0.5), (b.re - a.re) * Tc(0.5));
        }
        // xch becomes the next plane's row buffer; this plane's staging stage is refilled by the bulk-copy
        // engine (async proxy) after the generic reads above
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
    }
}

// Inverse: 2-D half spectra (T) -> real planes (T), out = x + add (add nullable).
template <typename T>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256, 1)
    k_plane_inv(const Cx<T>* __restrict__ spec, T* __restrict__ outp, const T* __restrict__ addp, int n3, int nitems,
                int64_t csf, int64_t css, int n1p, const Cx<T>* __restrict__ twx, const Cx<T>* __restrict__ twy) {
    using C = Plane2DCfg<T>;
    constexpr int N = C::N, L1 = C::L1, RPC = C::RPC, CPC = C::CPC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Cx<T>* buf0 = reinterpret_cast<Cx<T>*>(smem_raw);
    const unsigned r = cluster_rank(), cid = cluster_id(), ncl = cluster_count();
    const int la = threadIdx.x / C::TPLA, ta = threadIdx.x % C::TPLA;
    const int xb = threadIdx.x % CPC, tb = threadIdx.x / CPC;
    int it = 0;
    for (int item = (int)cid; item < nitems; item += (int)ncl, ++it) {
        const int st = it & 1;
        Cx<T>* rows = buf0 + (size_t)st * (C::BUFB / C::ES);
        Cx<T>* xch = buf0 + (size_t)(st ^ 1) * (C::BUFB / C::ES);
        const int comp = item / n3, z = item % n3;
        // phase B: inverse x2 FFT of column slot x; row p of the result goes to CTA p / 32
        const int x = (int)r * CPC + xb;
        const Cx<T>* sp = spec + comp * css + (int64_t)z * N * n1p;
        fft_line_io<T, N, +1, false, false>(xch + xb * C::LPB, tb, twy, 1, SpecColLd<T>{sp + x, n1p, x == 0 ? L1 : 0},
                                            PeerColSt<T>{rows, x});
        cluster_sync_all();
        // phase A: c2r along x1 of row 32r + la, + add
        Cx<T>* ln = rows + la * C::LPA;
        for (int k = ta; k <= L1 / 2; k += C::TPLA) {
            Cx<T> xk, xl;
            if (k == 0) {
                const Cx<T> zz = ln[P(0)];
                xk = cx(zz.re, T(0));
                xl = cx(zz.im, T(0));
            } else {
                xk = ln[P(k)];
                xl = ln[P(L1 - k)];
            }
            Cx<T> Zk, Zl;
            c2r_pair(xk, xl, twx[k], Zk, Zl);
            ln[P(k)] = Zk;
            if (k != 0 && 2 * k != L1) ln[P(L1 - k)] = Zl;
        }
        __syncthreads();
        const int64_t row = (int64_t)z * N + r * RPC + la;
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(outp + comp * csf) + row * L1;
        const Cx<T>* add = addp ? reinterpret_cast<const Cx<T>*>(addp + comp * csf) + row * L1 : nullptr;
        fft_line_io<T, L1, +1, true, false>(ln, ta, twx, 2, SmemLine<T>{ln}, RowSt<T>{dst, add, 0, true});
        __syncthreads();  // the row buffer is the next plane's exchange buffer
    }
}

template <typename Ti, typename Tc>
constexpr size_t plane_fwd_smem() {
    using C = Plane2DCfg<Tc>;
    constexpr int SI = staged_stride<Ti, C::TPLA>(C::L1) * (int)sizeof(Cx<Ti>);
    return 128 + 2 * (size_t)C::RPC * SI + 2 * C::BUFB + C::N * C::ES;
}
template <typename T>
constexpr size_t plane_inv_smem() {
    return 2 * Plane2DCfg<T>::BUFB;
}

}  // namespace dr
