// fft.cuh -- shared-memory Stockham FFT passes for the spectral operators (§III-B1,
// L303 §III-C1).  Every pass streams a field once from HBM into shared memory (16/8-byte cp.async,
// all of a CTA's loads in flight at once), transforms whole lines there (register butterflies of
// radix 16 in fp32 / radix 8 in fp64, padded smem against bank conflicts, twiddles from tables built
// in double precision on the host) and streams it back.
//
// Pass kinds
//   row_deriv      real rows (x1) -> d/dx1 (r2c, i k'_1, c2r), one HBM read + one write
//   col_deriv      real field read as complex pairs of adjacent x1 columns; d/dx2 or d/dx3 along
//                  strided lines (the multiplier i k' is Hermitian, so pairing is exact)
//   row_r2c / row_c2r   real rows <-> half-spectrum rows (padded row stride n1p)
//   col_fft        complex lines of a spectrum along x2 (forward or inverse)
//   col_middle     x3 lines of NCI spectra: forward FFT, pointwise symbol (NCI -> NCO), inverse FFT
// Normalisation: forward transforms are unnormalised; every symbol carries the inverse factor.
#pragma once
#include "common.cuh"

namespace dr {

// padded shared-memory index: one pad slot every 16 complex values
__device__ __forceinline__ int P(int i) { return i + (i >> 4); }
template <int L>
struct LineGeom {
    static constexpr int LP = L + L / 16 + 2;  // padded line length (holds index L for r2c)
};
// Threads per line: each owns the 16 values of one radix-16 butterfly per stage.
template <int L, typename T>
struct Tpl {
    static constexpr int R = 16;
    static constexpr int V = (L >= R) ? L / R : 1;
};
template <typename T>
struct CtaThreads {  // fp64 passes: fewer threads per CTA (large register footprint), more CTAs per SM
    static constexpr int V = sizeof(T) == 8 ? 128 : 256;
};
// Minimum resident CTAs of a pass for __launch_bounds__: 3 x 256 threads for fp32 compute (<= 80
// registers); 3 x 128 for fp64 (<= 170 registers for the radix-16 fp64 butterflies).
template <typename T, int NT>
struct MinB {
    static constexpr int V = sizeof(T) == 8 ? ((384 / NT) > 0 ? 384 / NT : 1) : ((768 / NT) > 0 ? 768 / NT : 1);
};
// Row passes: RB rows per CTA of ~256 threads.  Ti = type of the staged input when it differs from
// the compute type Tc (fp32 rows converted to fp64 in shared memory), else Ti = Tc.
template <int L, typename Tc, typename Ti = Tc>
struct RowCfg {
    static constexpr int TPL = Tpl<L, Tc>::V;
    static constexpr int RB = (CtaThreads<Tc>::V / TPL) > 0 ? CtaThreads<Tc>::V / TPL : 1;
    static constexpr int NT = RB * TPL;
    static constexpr size_t SMEM = (size_t)RB * LineGeom<L>::LP *
                                   (sizeof(Cx<Tc>) + (sizeof(Ti) != sizeof(Tc) ? sizeof(Cx<Ti>) : 0));
};

template <typename C>
__device__ __forceinline__ void cp_async_elem(C* smem, const C* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (sizeof(C) == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_join() {
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
}

// e^{DIR * 2 pi i m / 16}, m compile-time after unrolling
template <typename T, int DIR>
__device__ __forceinline__ Cx<T> w16(int m) {
    const double c[16] = {1.0, 0.92387953251128673848, 0.70710678118654752440, 0.38268343236508977173,
                          0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128673848,
                          -1.0, -0.92387953251128673848, -0.70710678118654752440, -0.38268343236508977173,
                          0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128673848};
    const double s[16] = {0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128673848,
                          1.0, 0.92387953251128673848, 0.70710678118654752440, 0.38268343236508977173,
                          0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128673848,
                          -1.0, -0.92387953251128673848, -0.70710678118654752440, -0.38268343236508977173};
    return cx<T>((T)c[m & 15], (T)(DIR * s[m & 15]));
}

// In-register DFT of length R (power of two <= 16), natural order in and out:
// X_k = sum_n x_n e^{DIR 2 pi i n k / R}.  Radix-2 decimation in time, twiddles constant-folded.
template <typename T, int R, int DIR>
struct DFT {
    static __device__ __forceinline__ void run(Cx<T>* x) {
        Cx<T> e[R / 2], o[R / 2];
#pragma unroll
        for (int i = 0; i < R / 2; ++i) { e[i] = x[2 * i]; o[i] = x[2 * i + 1]; }
        DFT<T, R / 2, DIR>::run(e);
        DFT<T, R / 2, DIR>::run(o);
#pragma unroll
        for (int k = 0; k < R / 2; ++k) {
            const int m = k * (16 / R);
            Cx<T> t;
            if (m == 0) t = o[k];
            else if (m == 4) t = (DIR < 0) ? cx(o[k].im, -o[k].re) : cx(-o[k].im, o[k].re);
            else t = cmul(o[k], w16<T, DIR>(m));
            x[k] = e[k] + t;
            x[k + R / 2] = e[k] - t;
        }
    }
};
template <typename T, int DIR>
struct DFT<T, 1, DIR> {
    static __device__ __forceinline__ void run(Cx<T>*) {}
};

// One Stockham autosort stage of radix R (Ns = product of the previous radices) on a line of
// length L held in padded shared memory.  Each of the TPL threads of the line owns NB = L/R/TPL
// butterflies.  tw: table of e^{-2 pi i m / (L*tws)}, m < L*tws.
template <typename T, int L, int R, int Ns, int DIR, int TPL>
__device__ __forceinline__ void stockham_stage(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws) {
    constexpr int NB = (L / R) / TPL;
    Cx<T> x[NB][R];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = t + b * TPL;
#pragma unroll
        for (int r = 0; r < R; ++r) x[b][r] = buf[P(j + r * (L / R))];
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = t + b * TPL;
        const int k = j & (Ns - 1);
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const int m = r * k * (L / (Ns * R));
                Cx<T> w = tw[m * tws];
                if (DIR > 0) w.im = -w.im;
                x[b][r] = cmul(x[b][r], w);
            }
        }
        DFT<T, R, DIR>::run(x[b]);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[P(base + r * Ns)] = x[b][r];
    }
    __syncthreads();
}

template <typename T, int L, int DIR, int TPL, int R, int Ns>
__device__ __forceinline__ void fft_stages(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws) {
    if constexpr (Ns * R >= L) {
        stockham_stage<T, L, L / Ns, Ns, DIR, TPL>(buf, t, tw, tws);
    } else {
        stockham_stage<T, L, R, Ns, DIR, TPL>(buf, t, tw, tws);
        fft_stages<T, L, DIR, TPL, R, Ns * R>(buf, t, tw, tws);
    }
}

// Whole-line FFT (in place, padded layout), radix plan R x R x ... x r with R = 16 (fp32) / 8 (fp64).
// Every thread of the CTA must call this (it contains __syncthreads).
template <typename T, int L, int DIR>
__device__ __forceinline__ void fft_line(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws) {
    fft_stages<T, L, DIR, Tpl<L, T>::V, Tpl<L, T>::R, 1>(buf, t, tw, tws);
}

// ---------------------------------------------------------------------------------------------
// real <-> half-complex post/pre-processing of a row of N = 2L reals packed as L complex
// z_n = x_{2n} + i x_{2n+1}.  After the forward L-point FFT Z, X_k (k = 0..L) of the N-point DFT:
//   E = (Z_k + conj Z_{L-k})/2, O = (Z_k - conj Z_{L-k})/(2i), X_k = E + W^k O, X_{L-k} = conj(E - W^k O),
// W = e^{-2 pi i/N}.  Pairs (k, L-k) are handled by one thread, so the update is in place.
template <typename T, int L, int TPL>
__device__ __forceinline__ void r2c_post(Cx<T>* buf, int t, const Cx<T>* __restrict__ twN) {
    for (int k = t; k <= L / 2; k += TPL) {
        const Cx<T> zk = buf[P(k)];
        const Cx<T> zl = buf[P(k == 0 ? 0 : L - k)];
        const Cx<T> E = cx((zk.re + zl.re) * T(0.5), (zk.im - zl.im) * T(0.5));
        // (Z_k - conj Z_{L-k}) / (2i) = (a + ib)/(2i) = (b - ia)/2 with a + ib = Z_k - conj Z_{L-k}
        const T a = zk.re - zl.re, b = zk.im + zl.im;
        const Cx<T> O = cx(b * T(0.5), -a * T(0.5));
        const Cx<T> WO = cmul(twN[k], O);
        const Cx<T> Xk = E + WO;
        const Cx<T> Xl = conj(E - WO);
        buf[P(k)] = Xk;
        buf[P(L - k)] = Xl;  // k = 0 writes X_L into slot L; k = L/2 writes the same slot twice
    }
    __syncthreads();
}

// inverse: given X_0..X_L, Z_k = E + i O with E = (X_k + conj X_{L-k})/2,
// O = (X_k - conj X_{L-k}) conj(W^k)/2, and Z_{L-k} = conj(E) + i conj(O).
template <typename T, int L, int TPL>
__device__ __forceinline__ void c2r_pre(Cx<T>* buf, int t, const Cx<T>* __restrict__ twN) {
    for (int k = t; k <= L / 2; k += TPL) {
        const Cx<T> xk = buf[P(k)];
        const Cx<T> xl = buf[P(L - k)];
        const Cx<T> E = cx((xk.re + xl.re) * T(0.5), (xk.im - xl.im) * T(0.5));
        const Cx<T> D = cx((xk.re - xl.re) * T(0.5), (xk.im + xl.im) * T(0.5));
        const Cx<T> O = cmul(D, conj(twN[k]));
        buf[P(k)] = cx(E.re - O.im, E.im + O.re);            // E + iO
        if (k != 0 && 2 * k != L) buf[P(L - k)] = cx(E.re + O.im, -E.im + O.re);  // conj(E) + i conj(O)
    }
    __syncthreads();
}

// Stage RB contiguous rows of L complex values (row r of the CTA at src + r L) into padded lines
// sm + r LP, asynchronously, one complex value (8 or 16 bytes) per cp.async.
template <typename C, int L, int NT>
__device__ __forceinline__ void row_stage(C* sm, const C* __restrict__ src, int nvalid) {
    constexpr int LP = LineGeom<L>::LP;
    for (int e = threadIdx.x; e < nvalid * L; e += NT) cp_async_elem(sm + (e / L) * LP + P(e % L), src + e);
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// Driver shared by every FFT pass.  DB = true: persistent, a CTA walks tiles blockIdx.x, + gridDim.x,
// ... with two shared-memory buffers (the next tile's cp.async loads fly while the current tile is
// transformed and stored); DB = false: one tile per CTA, the hardware overlaps resident CTAs.
// PassT supplies NT, MINB, BUF (bytes per buffer), ntiles(), load(tile, smem), run(tile, smem).
template <class PassT, bool DB>
__global__ void __launch_bounds__(PassT::NT, PassT::MINB) k_stream(PassT pass) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int tile = blockIdx.x;
    const int ntiles = pass.ntiles();
    if (tile >= ntiles) return;
    if constexpr (!DB) {  // one tile per CTA: load, transform, store
        pass.load(tile, smem_raw);
        cp_async_join();
        pass.run(tile, smem_raw);
        return;
    }
    pass.load(tile, smem_raw);
    cp_async_commit();
    int cur = 0;
    for (;;) {
        const int next = tile + gridDim.x;
        const bool more = next < ntiles;
        if (more) pass.load(next, smem_raw + (cur ^ 1) * PassT::BUF);
        cp_async_commit();
        cp_async_wait1();  // everything but the newest group has landed: the current tile is in smem
        __syncthreads();
        pass.run(tile, smem_raw + cur * PassT::BUF);
        if (!more) break;
        __syncthreads();  // the current buffer is refilled by the next iteration's prefetch
        tile = next;
        cur ^= 1;
    }
}

// Row pass: x1-derivative of real rows ("N2 N3 1D FFTs across the first coordinate,
// diagonal scaling, and then the same number of inverse FFTs").  out = acc*out + d f/dx1.
template <typename T, int L>
struct RowDerivPass {
    using RC = RowCfg<L, T>;
    static constexpr int TPL = RC::TPL, LP = LineGeom<L>::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUF = (size_t)RB * LP * sizeof(Cx<T>);
    Grid g;
    const T* f;
    T* out;
    int accumulate;
    const Cx<T>* twN;
    __device__ __forceinline__ int ntiles() const { return (int)(((int64_t)g.n2 * g.n3 + RB - 1) / RB); }
    __device__ __forceinline__ int nvalid(int tile) const {
        const int64_t rem = (int64_t)g.n2 * g.n3 - (int64_t)tile * RB;
        return (int)(rem < RB ? rem : RB);
    }
    __device__ __forceinline__ void load(int tile, unsigned char* smem) const {
        row_stage<Cx<T>, L, NT>(reinterpret_cast<Cx<T>*>(smem), reinterpret_cast<const Cx<T>*>(f) + (int64_t)tile * RB * L,
                                nvalid(tile));
    }
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        const int nv = nvalid(tile);
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        Cx<T>* buf = sm + line * LP;
        fft_line<T, L, -1>(buf, t, twN, 2);
        r2c_post<T, L, TPL>(buf, t, twN);
        // X_k *= i k'_1 / L  (k = 0..L; Nyquist k = L is zeroed, reading A2; 1/L normalises the c2r)
        for (int k = t; k <= L; k += TPL) {
            const T kk = (k == L) ? T(0) : T(k);
            buf[P(k)] = mul_i(buf[P(k)], kk / T(L));
        }
        __syncthreads();
        c2r_pre<T, L, TPL>(buf, t, twN);
        fft_line<T, L, +1>(buf, t, twN, 2);
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(out) + (int64_t)tile * RB * L;
        for (int e = threadIdx.x; e < nv * L; e += NT) {
            Cx<T> v = sm[(e / L) * LP + P(e % L)];
            if (accumulate) { const Cx<T> o = dst[e]; v = v + o; }
            dst[e] = v;
        }
    }
};

// Row pass: real rows (type Ti) -> half-spectrum rows (r2c along x1) computed and stored in Tc,
// spectrum row stride g.n1p.  Ti = float, Tc = double keeps the forward spectrum exact enough for the
// high-wavenumber amplification of beta*A.
// The fp32 rows are staged asynchronously into their own buffer and widened in shared memory.
template <typename Ti, typename Tc, int L>
struct RowR2cPass {
    using RC = RowCfg<L, Tc, Ti>;
    static constexpr int TPL = RC::TPL, LP = LineGeom<L>::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<Tc, NT>::V;
    static constexpr size_t BUF = RC::SMEM;
    static constexpr size_t STG = (size_t)RB * LP * sizeof(Cx<Tc>);  // offset of the Ti staging lines
    Grid g;
    const Ti* f;
    Cx<Tc>* spec;
    const Cx<Tc>* twN;
    __device__ __forceinline__ int ntiles() const { return (int)(((int64_t)g.n2 * g.n3 + RB - 1) / RB); }
    __device__ __forceinline__ int nvalid(int tile) const {
        const int64_t rem = (int64_t)g.n2 * g.n3 - (int64_t)tile * RB;
        return (int)(rem < RB ? rem : RB);
    }
    __device__ __forceinline__ void load(int tile, unsigned char* smem) const {
        const Cx<Ti>* src = reinterpret_cast<const Cx<Ti>*>(f) + (int64_t)tile * RB * L;
        if constexpr (sizeof(Ti) == sizeof(Tc)) row_stage<Cx<Tc>, L, NT>(reinterpret_cast<Cx<Tc>*>(smem), reinterpret_cast<const Cx<Tc>*>(src), nvalid(tile));
        else row_stage<Cx<Ti>, L, NT>(reinterpret_cast<Cx<Ti>*>(smem + STG), src, nvalid(tile));
    }
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<Tc>* sm = reinterpret_cast<Cx<Tc>*>(smem);
        const int nv = nvalid(tile);
        if constexpr (sizeof(Ti) != sizeof(Tc)) {
            const Cx<Ti>* st = reinterpret_cast<const Cx<Ti>*>(smem + STG);
            for (int e = threadIdx.x; e < nv * L; e += NT) {
                const int o = (e / L) * LP + P(e % L);
                const Cx<Ti> v = st[o];
                sm[o] = cx<Tc>((Tc)v.re, (Tc)v.im);
            }
            __syncthreads();
        }
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        Cx<Tc>* buf = sm + line * LP;
        fft_line<Tc, L, -1>(buf, t, twN, 2);
        r2c_post<Tc, L, TPL>(buf, t, twN);
        constexpr int NC = L + 1;
        const int64_t row0 = (int64_t)tile * RB;
        for (int e = threadIdx.x; e < nv * NC; e += NT) {
            const int r = e / NC, k = e % NC;
            spec[(row0 + r) * g.n1p + k] = sm[r * LP + P(k)];
        }
    }
};

// Row pass epilogue for the c2r inverse: out = x (+ add)
template <typename T>
struct RowOut {
    T* out;
    const T* add;  // nullable: field added after the inverse (b~ in the non-isochoric matvec)
};

// Row pass: half-spectrum rows -> real rows (c2r along x1) in T with epilogue out = x + add.
// The spectrum already carries the full inverse normalisation.
template <typename T, int L>
struct RowC2rPass {
    using RC = RowCfg<L, T>;
    static constexpr int TPL = RC::TPL, LP = LineGeom<L>::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUF = (size_t)RB * LP * sizeof(Cx<T>);
    Grid g;
    const Cx<T>* spec;
    RowOut<T> epi;
    const Cx<T>* twN;
    __device__ __forceinline__ int ntiles() const { return (int)(((int64_t)g.n2 * g.n3 + RB - 1) / RB); }
    __device__ __forceinline__ int nvalid(int tile) const {
        const int64_t rem = (int64_t)g.n2 * g.n3 - (int64_t)tile * RB;
        return (int)(rem < RB ? rem : RB);
    }
    __device__ __forceinline__ void load(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        constexpr int NC = L + 1;
        const int64_t row0 = (int64_t)tile * RB;
        const int nv = nvalid(tile);
        for (int e = threadIdx.x; e < nv * NC; e += NT) {
            const int r = e / NC, k = e % NC;
            cp_async_elem(sm + r * LP + P(k), spec + (row0 + r) * g.n1p + k);
        }
    }
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        const int nv = nvalid(tile);
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        Cx<T>* buf = sm + line * LP;
        c2r_pre<T, L, TPL>(buf, t, twN);
        fft_line<T, L, +1>(buf, t, twN, 2);
        const int64_t row0 = (int64_t)tile * RB;
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(epi.out) + row0 * L;
        const Cx<T>* add = epi.add ? reinterpret_cast<const Cx<T>*>(epi.add) + row0 * L : nullptr;
        for (int e = threadIdx.x; e < nv * L; e += NT) {
            Cx<T> v = sm[(e / L) * LP + P(e % L)];
            if (add) v = v + add[e];
            dst[e] = v;
        }
    }
};

// ---------------------------------------------------------------------------------------------
// Column passes along x2 (AX = 2) or x3 (AX = 3) of a complex array with W complex columns per row
// (W = n1p for spectra, N1/2 for a real field read as pairs) and extents (W, n2, n3).
// A CTA owns XC consecutive columns x OL lines of the other transverse axis.
struct ColGeom {
    int W;      // row stride in complex elements
    int nx;     // valid columns (x < nx)
    int n2, n3;
    int k2off = 0, n2g = 0;  // slab transposes: global x2 index = local + k2off, global extent n2g
};

// "Split" layout of a slab's spectrum (multi-GPU x2 passes): the x2 extent is cut into blocks of nb
// lines, block q destined to / received from rank q, stored as [q][i3][i2 % nb][x] so every rank's
// chunk of an all-to-all transpose is contiguous.  nb = 0: the plain [i3][i2][x] layout.
template <int AX>
__device__ __forceinline__ int64_t col_addr(const ColGeom& c, int x, int other, int p, int nb = 0) {
    if (AX == 2) {
        if (nb) return ((((int64_t)(p / nb) * c.n3 + other) * nb) + (p % nb)) * c.W + x;
        return ((int64_t)other * c.n2 + p) * c.W + x;  // other = i3, p = i2
    }
    return ((int64_t)p * c.n2 + other) * c.W + x;      // other = i2, p = i3
}

// CTA shape of a column pass: XC columns (one 128-byte segment: 16 complex64 / 8 complex128) x OL
// transverse lines, TPL threads per line, ~256 threads, capped so NC components of the CTA's lines
// fit in ~96 KB of shared memory.
template <int L, typename T, int NC = 1>
struct ColCfg {
    static constexpr int ES = (int)sizeof(Cx<T>);
    static constexpr int TPL = Tpl<L, T>::V;
    static constexpr int LPB = LineGeom<L>::LP * ES;  // bytes per line
    static constexpr int XC0 = 128 / ES;
    static constexpr int XC = (NC * XC0 * LPB <= 96 * 1024) ? XC0 : (NC * (XC0 / 2) * LPB <= 96 * 1024) ? XC0 / 2 : XC0 / 4;
    static constexpr int OLT = (XC * TPL >= CtaThreads<T>::V) ? 1 : CtaThreads<T>::V / (XC * TPL);
    static constexpr int MAXL = (96 * 1024) / (NC * LPB);
    static constexpr int OLS = (MAXL / XC) >= 1 ? MAXL / XC : 1;
    static constexpr int OL = OLT < OLS ? OLT : OLS;
    static constexpr int NT = XC * OL * TPL;
    static constexpr int LINES = XC * OL;
    static constexpr size_t SMEM = (size_t)NC * LINES * LineGeom<L>::LP * ES;
};

template <typename T, int L, int XC, int OL, int AX, int NT>
__device__ __forceinline__ void col_load(Cx<T>* sm, const Cx<T>* __restrict__ src, const ColGeom& c, int x0, int o0,
                                         int nother, int nb = 0) {
    constexpr int LP = LineGeom<L>::LP;
    for (int e = threadIdx.x; e < XC * L * OL; e += NT) {
        const int xi = e % XC, p = (e / XC) % L, oi = e / (XC * L);
        const int x = x0 + xi, o = o0 + oi;
        Cx<T>* d = sm + (oi * XC + xi) * LP + P(p);
        if (x < c.nx && o < nother) cp_async_elem(d, src + col_addr<AX>(c, x, o, p, nb));
        else *d = cx(T(0), T(0));
    }
}

template <typename T, int L, int XC, int OL, int AX, bool ACC, int NT, typename To = T>
__device__ __forceinline__ void col_store(const Cx<T>* sm, Cx<To>* __restrict__ dst, const ColGeom& c, int x0, int o0,
                                          int nother, int nb = 0) {
    constexpr int LP = LineGeom<L>::LP;
    for (int e = threadIdx.x; e < XC * L * OL; e += NT) {
        const int xi = e % XC, p = (e / XC) % L, oi = e / (XC * L);
        const int x = x0 + xi, o = o0 + oi;
        if (x < c.nx && o < nother) {
            const Cx<T> w = sm[(oi * XC + xi) * LP + P(p)];
            Cx<To> v = cx<To>((To)w.re, (To)w.im);
            const int64_t a = col_addr<AX>(c, x, o, p, nb);
            if (ACC) v = v + dst[a];
            dst[a] = v;
        }
    }
}

// Derivative along x2 / x3 of a real field (viewed as complex pairs): out (+)= d f / dx_AX.
template <typename T, int L, int AX>
struct ColDerivPass {
    using CC = ColCfg<L, T>;
    static constexpr int TPL = CC::TPL, LP = LineGeom<L>::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUF = CC::SMEM;
    ColGeom c;
    const Cx<T>* src;
    Cx<T>* dst;
    int accumulate;
    const Cx<T>* tw;
    __device__ __forceinline__ int nother() const { return (AX == 2) ? c.n3 : c.n2; }
    __device__ __forceinline__ int ntiles() const { return ((c.nx + XC - 1) / XC) * ((nother() + OL - 1) / OL); }
    __device__ __forceinline__ void origin(int tile, int& x0, int& o0) const {
        const int nxb = (c.nx + XC - 1) / XC;
        x0 = (tile % nxb) * XC;
        o0 = (tile / nxb) * OL;
    }
    __device__ __forceinline__ void load(int tile, unsigned char* smem) const {
        int x0, o0;
        origin(tile, x0, o0);
        col_load<T, L, XC, OL, AX, NT>(reinterpret_cast<Cx<T>*>(smem), src, c, x0, o0, nother());
    }
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        int x0, o0;
        origin(tile, x0, o0);
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        Cx<T>* buf = sm + line * LP;
        fft_line<T, L, -1>(buf, t, tw, 1);
        for (int k = t; k < L; k += TPL) {
            const T kp = (T)wavenum_odd(k, L);
            buf[P(k)] = mul_i(buf[P(k)], kp / T(L));
        }
        __syncthreads();
        fft_line<T, L, +1>(buf, t, tw, 1);
        if (accumulate) col_store<T, L, XC, OL, AX, true, NT>(sm, dst, c, x0, o0, nother());
        else col_store<T, L, XC, OL, AX, false, NT>(sm, dst, c, x0, o0, nother());
    }
};

// Complex FFT of spectrum columns along x2 (forward DIR=-1 or inverse DIR=+1), src -> dst (may alias
// when both layouts are plain).  nb_in / nb_out != 0 select the split layout on that side (the
// all-to-all chunks of the multi-GPU transposes), fusing the pack / unpack into this pass.
template <typename T, int L, int DIR>
struct ColFftPass {
    using CC = ColCfg<L, T>;
    static constexpr int TPL = CC::TPL, LP = LineGeom<L>::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUF = CC::SMEM;
    ColGeom c;
    const Cx<T>* src;
    Cx<T>* dst;
    const Cx<T>* tw;
    int nb_in, nb_out;
    __device__ __forceinline__ int ntiles() const { return ((c.nx + XC - 1) / XC) * ((c.n3 + OL - 1) / OL); }
    __device__ __forceinline__ void origin(int tile, int& x0, int& o0) const {
        const int nxb = (c.nx + XC - 1) / XC;
        x0 = (tile % nxb) * XC;
        o0 = (tile / nxb) * OL;
    }
    __device__ __forceinline__ void load(int tile, unsigned char* smem) const {
        int x0, o0;
        origin(tile, x0, o0);
        col_load<T, L, XC, OL, 2, NT>(reinterpret_cast<Cx<T>*>(smem), src, c, x0, o0, c.n3, nb_in);
    }
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        int x0, o0;
        origin(tile, x0, o0);
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        fft_line<T, L, DIR>(sm + line * LP, t, tw, 1);
        col_store<T, L, XC, OL, 2, false, NT>(sm, dst, c, x0, o0, c.n3, nb_out);
    }
};

// ---------------------------------------------------------------------------------------------
// Spectral symbols applied in the x3 middle pass.  k = (k1, k2, k3) signed wavenumbers,
// kp = (k1', k2', k3') with the Nyquist zeroed.  `norm` = full inverse normalisation 2/M.
struct SymInfo {
    int reg;       // 1: a = |k|^2, 2: a = |k|^4
    double beta;
    double norm;
};

template <typename T>
__device__ __forceinline__ T sym_a(const SymInfo& s, T kk) { return s.reg == 1 ? kk : kk * kk; }

// kind 0: Y = norm * beta a(k) X                  (regulariser, Eq. 5e)
// kind 1: Y = norm * X / (beta a_hat(k))          (preconditioner; a_hat(0) = 1)
// kind 2: Y = norm * L_hat X                      (Leray, 3 -> 3)
// kind 3: Y = norm * L_hat X / (beta a_hat(k))    (isochoric preconditioner)
// kind 4: Y = norm * (beta a(k) V + L_hat B)      (isochoric matvec tail, 6 -> 3)
template <typename T, int KIND>
struct Sym {
    static constexpr int NCI = (KIND <= 1) ? 1 : (KIND == 4 ? 6 : 3);
    static constexpr int NCO = (KIND <= 1) ? 1 : 3;
    static __device__ __forceinline__ void apply(const SymInfo& s, Cx<T>* x, int k1, int k2, int k3, int kp1, int kp2,
                                                 int kp3) {
        const T kk = T(k1) * T(k1) + T(k2) * T(k2) + T(k3) * T(k3);
        const T nrm = (T)s.norm;
        if (KIND == 0) {
            x[0] = scale(x[0], nrm * (T)s.beta * sym_a<T>(s, kk));
        } else if (KIND == 1) {
            const T ah = (kk == T(0)) ? T(1) : sym_a<T>(s, kk);
            x[0] = scale(x[0], nrm / ((T)s.beta * ah));
        } else {
            const T q1 = T(kp1), q2 = T(kp2), q3 = T(kp3);
            const T qq = q1 * q1 + q2 * q2 + q3 * q3;
            Cx<T>* B = (KIND == 4) ? x + 3 : x;
            Cx<T> b0 = B[0], b1 = B[1], b2 = B[2];
            if (qq != T(0)) {
                const T inv = T(1) / qq;
                const Cx<T> kd = cx((q1 * b0.re + q2 * b1.re + q3 * b2.re) * inv, (q1 * b0.im + q2 * b1.im + q3 * b2.im) * inv);
                b0 = b0 - scale(kd, q1);
                b1 = b1 - scale(kd, q2);
                b2 = b2 - scale(kd, q3);
            }
            T f = nrm;
            if (KIND == 3) f = nrm / ((T)s.beta * ((kk == T(0)) ? T(1) : sym_a<T>(s, kk)));
            if (KIND == 4) {
                const T ra = nrm * (T)s.beta * sym_a<T>(s, kk);
                x[0] = scale(x[0], ra) + scale(b0, nrm);
                x[1] = scale(x[1], ra) + scale(b1, nrm);
                x[2] = scale(x[2], ra) + scale(b2, nrm);
            } else {
                x[0] = scale(b0, f);
                x[1] = scale(b1, f);
                x[2] = scale(b2, f);
            }
        }
    }
};

template <typename T, int NC>
struct SpecPtrs {
    Cx<T>* p[NC];
};

// x3 middle pass: forward FFT of NCI spectra along x3 in Ti, symbol in Ti, then the NCO results are
// narrowed to To in a second shared-memory region and transformed back in To (the inverse passes after
// the symbol may run in the I/O precision: their rounding is relative to the already-amplified signal).
template <typename Ti, typename To, int L, int KIND>
struct MiddlePass {
    using T = Ti;
    static constexpr int NCI = Sym<T, KIND>::NCI, NCO = Sym<T, KIND>::NCO;
    using CC = ColCfg<L, T, NCI>;
    static constexpr int TPL = CC::TPL, LP = LineGeom<L>::LP, XC = CC::XC, OL = CC::OL, LINES = CC::LINES, NT = CC::NT;
    static_assert(Tpl<L, To>::V == TPL, "inverse lines use the same threads");
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUFI = CC::SMEM;
    static constexpr size_t BUF = BUFI + (size_t)NCO * LINES * LP * sizeof(Cx<To>);
    ColGeom c;
    SpecPtrs<Ti, NCI> in;
    SpecPtrs<To, NCO> out;
    SymInfo s;
    const Cx<Ti>* tw;
    const Cx<To>* two;  // inverse twiddles in To
    __device__ __forceinline__ int ntiles() const { return ((c.nx + XC - 1) / XC) * ((c.n2 + OL - 1) / OL); }
    __device__ __forceinline__ void origin(int tile, int& x0, int& o0) const {
        const int nxb = (c.nx + XC - 1) / XC;
        x0 = (tile % nxb) * XC;
        o0 = (tile / nxb) * OL;
    }
    __device__ __forceinline__ void load(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        int x0, o0;
        origin(tile, x0, o0);
#pragma unroll
        for (int ci = 0; ci < NCI; ++ci) col_load<T, L, XC, OL, 3, NT>(sm + ci * LINES * LP, in.p[ci], c, x0, o0, c.n2);
    }
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        Cx<To>* so = reinterpret_cast<Cx<To>*>(smem + BUFI);
        int x0, o0;
        origin(tile, x0, o0);
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
#pragma unroll
        for (int ci = 0; ci < NCI; ++ci) fft_line<T, L, -1>(sm + ci * LINES * LP + line * LP, t, tw, 1);
        // symbol: element (line, p): k1 = column index x (0..N1/2), k2 from the transverse index, k3 from p
        const int n1 = 2 * (c.nx - 1);
        for (int e = threadIdx.x; e < LINES * L; e += NT) {
            const int ln = e / L, p = e % L;
            const int xi = ln % XC, oi = ln / XC;
            const int x = x0 + xi, o = o0 + oi;
            Cx<T> v[NCI];
#pragma unroll
            for (int ci = 0; ci < NCI; ++ci) v[ci] = sm[ci * LINES * LP + ln * LP + P(p)];
            if (x < c.nx && o < c.n2) {
                const int og = o + c.k2off, n2g = c.n2g ? c.n2g : c.n2;
                const int k1 = x, k2 = wavenum(og, n2g), k3 = wavenum(p, L);
                const int kp1 = (x == n1 / 2) ? 0 : x, kp2 = wavenum_odd(og, n2g), kp3 = wavenum_odd(p, L);
                Sym<T, KIND>::apply(s, v, k1, k2, k3, kp1, kp2, kp3);
            }
#pragma unroll
            for (int co = 0; co < NCO; ++co) so[co * LINES * LP + ln * LP + P(p)] = cx<To>((To)v[co].re, (To)v[co].im);
        }
        __syncthreads();
#pragma unroll
        for (int co = 0; co < NCO; ++co) fft_line<To, L, +1>(so + co * LINES * LP + line * LP, t, two, 1);
#pragma unroll
        for (int co = 0; co < NCO; ++co)
            col_store<To, L, XC, OL, 3, false, NT, To>(so + co * LINES * LP, out.p[co], c, x0, o0, c.n2);
    }
};

}  // namespace dr
