// fft.cuh -- Stockham FFT passes for the spectral operators (§III-B1, L303 §III-C1).
// Every pass streams a field once through the SM: the first radix-16 stage of a line reads its 16
// operands straight from global memory into registers (coalesced: consecutive lanes read consecutive
// addresses), the stages in between exchange through padded shared memory, and the last stage writes
// its results straight to global memory in natural order -- one shared-memory round trip per stage
// boundary instead of staging whole lines in and out.  Register butterflies of radix 16 with
// constant-folded inner twiddles; stage twiddles from tables built in double precision on the host.
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
#include <cuda.h>  // CUtensorMap (the tensor map is encoded on the host through the runtime's driver entry point)
#include "common.cuh"

namespace dr {

// padded shared-memory index: one pad slot every 16 complex values
__device__ __forceinline__ int P(int i) { return i + (i >> 4); }
// Padded line stride in complex elements: the smallest LP >= P(L) + 1 (holds index L for r2c) with
// LP = REM (mod MOD).  The stride is chosen per pass from how the lanes of one shared-memory wavefront
// (128 bytes: W = 128 / sizeof(Cx<T>) lanes) spread over lines, so that they hit distinct banks.
// Within a line, the lane with thread-in-line index t sits at element offset t (mod 16) in every stage
// (P pads one slot per 16), so
//   row passes (TPL consecutive lanes per line, W / TPL lines per wavefront): LP = TPL (mod W);
//   column passes (XC consecutive lanes = columns, each its own line, W / XC values of t per
//   wavefront): LP = max(1, W / XC) (mod W).
template <int L, int MOD, int REM>
struct PadLP {
    static constexpr int B = L + L / 16 + 1;
    static constexpr int V = (MOD <= 1) ? B : B + (((REM - B) % MOD) + MOD) % MOD;
};
template <typename T>
struct WaveLanes {  // lanes of one 128-byte shared-memory wavefront for complex T
    static constexpr int V = 128 / (int)(2 * sizeof(T));
};
template <int L, typename T, int TPL>
struct RowLP {
    static constexpr int W = WaveLanes<T>::V;
    static constexpr int V = (TPL < W) ? PadLP<L, W, TPL>::V : PadLP<L, 1, 0>::V;
};
template <int L, typename T, int XC>
struct ColLP {
    static constexpr int W = WaveLanes<T>::V;
    static constexpr int V = PadLP<L, W, (XC >= W) ? 1 : W / XC>::V;
};
// Threads per line: each owns the 16 values of one radix-16 butterfly per stage.
template <int L, typename T>
struct Tpl {
    static constexpr int R = 16;  // (radix 8 for fp64 halves the registers but adds a shared-memory exchange: slower)
    static constexpr int V = (L >= R) ? L / R : 1;
};
template <typename T>
struct CtaThreads {  // fp64 passes: fewer threads per CTA (large register footprint), more CTAs per SM
    static constexpr int V = sizeof(T) == 8 ? 128 : 256;
};
// Minimum resident CTAs of a pass for __launch_bounds__: 3 x 256 threads for fp32 compute (<= 80
// registers); 4 x 128 for fp64 (<= 128 registers for the radix-16 fp64 butterflies), 3 x 128 for the
// fp64 middle pass (measured: r2c 67 -> 64 us at 128 registers, middle 88 -> 92 us).
template <typename T, int NT>
struct MinB {
    static constexpr int V = sizeof(T) == 8 ? ((512 / NT) > 0 ? 512 / NT : 1) : ((768 / NT) > 0 ? 768 / NT : 1);
};
template <typename T, int NT>
struct MinBMiddle {  // the x3 middle pass keeps 160 registers in fp64 (forward + symbol + fp32 inverse)
    static constexpr int V = sizeof(T) == 8 ? ((384 / NT) > 0 ? 384 / NT : 1) : ((768 / NT) > 0 ? 768 / NT : 1);
};
// Row passes: RB rows per CTA.
template <int L, typename Tc>
struct RowCfg {
    static constexpr int TPL = Tpl<L, Tc>::V;
    static constexpr int RB = (CtaThreads<Tc>::V / TPL) > 0 ? CtaThreads<Tc>::V / TPL : 1;
    static constexpr int NT = RB * TPL;
    static constexpr int LP = RowLP<L, Tc, TPL>::V;
    static constexpr size_t SMEM = (size_t)RB * LP * sizeof(Cx<Tc>);
};

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

// ---------------------------------------------------------------------------------------------
// Line accessors: element i (0 <= i < L) of the line a thread works on.
template <typename T>
struct SmemLine {
    Cx<T>* b;
    __device__ __forceinline__ Cx<T> ld(int i) const { return b[P(i)]; }
    __device__ __forceinline__ void st(int i, const Cx<T>& v) const { b[P(i)] = v; }
};

// Stage-major twiddle table (tws < 0 in stage_io): for every stage with Ns > 1 and radix Rs, the
// entries w(r, k) = e^{DIR 2 pi i r k / (Ns Rs)} for r = 1..Rs-1, k = 0..Ns-1 stored as [r - 1][k], so
// the lanes of a line (consecutive k) read consecutive entries.  The natural table indexed by
// m = r k L / (Ns Rs) put those lanes r * L / (Ns Rs) entries apart: up to 8-way shared-memory bank
// conflicts on 16-byte complex128 entries (ncu: the fp64 staged r2c pass at 1.61 wavefronts per LDS).
// Offset of stage Ns in the table of a radix-R plan of length L (R = 16, last radix L / Ns):
template <int L, int R>
__host__ __device__ constexpr int stage_tw_off(int Ns) {
    int off = 0;
    for (int n = R; n < Ns; n *= R) off += ((L / n < R ? L / n : R) - 1) * n;
    return off;
}
template <int L, int R>
__host__ __device__ constexpr int stage_tw_count() {
    int n = R;
    while (n < L) n *= R;
    return stage_tw_off<L, R>(n);
}

// One Stockham autosort stage of radix R (Ns = product of the previous radices) on a line of length L.
// Each of the TPL threads of the line owns NB = L/R/TPL butterflies; operands come from src.ld, results
// go to dst.st (shared memory or global).  SYNC: the stage is in place in shared memory, so all reads
// must finish (barrier) before the writes.  tw: table of e^{-2 pi i m / (L*tws)}, m < L*tws; tws < 0:
// the stage-major table above (of the line's radix-16 plan).
template <typename T, int L, int R, int Ns, int DIR, int TPL, bool SYNC, class Src, class Dst>
__device__ __forceinline__ void stage_io(int t, const Cx<T>* __restrict__ tw, int tws, const Src& src, const Dst& dst) {
    constexpr int NB = (L / R) / TPL;
    Cx<T> x[NB][R];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = t + b * TPL;
#pragma unroll
        for (int r = 0; r < R; ++r) x[b][r] = src.ld(j + r * (L / R));
    }
    if (SYNC) __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = t + b * TPL;
        const int k = j & (Ns - 1);
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const int m = r * k * (L / (Ns * R));
                Cx<T> w = tws < 0 ? tw[stage_tw_off<L, 16>(Ns) + (r - 1) * Ns + k] : tw[m * tws];
                if (DIR > 0) w.im = -w.im;
                x[b][r] = cmul(x[b][r], w);
            }
        }
        DFT<T, R, DIR>::run(x[b]);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst.st(base + r * Ns, x[b][r]);
    }
}

// stages Ns, Ns*R, ... of a line whose data sit in shared memory `buf`; the last stage writes to dst
template <typename T, int L, int DIR, int TPL, int R, int Ns, bool DST_SMEM, class Dst>
__device__ __forceinline__ void stages_rest(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws, const Dst& dst) {
    if constexpr (Ns * R >= L) {
        stage_io<T, L, L / Ns, Ns, DIR, TPL, DST_SMEM>(t, tw, tws, SmemLine<T>{buf}, dst);
        if (DST_SMEM) __syncthreads();
    } else {
        stage_io<T, L, R, Ns, DIR, TPL, true>(t, tw, tws, SmemLine<T>{buf}, SmemLine<T>{buf});
        __syncthreads();
        stages_rest<T, L, DIR, TPL, R, Ns * R, DST_SMEM>(buf, t, tw, tws, dst);
    }
}

// Whole-line FFT, radix plan R x R x ... x r (R = 16 fp32, 8 fp64): src -> [shared line buf] -> dst.  SRC_SMEM / DST_SMEM:
// the source / destination is `buf` itself (in place).  Every thread of the CTA must call this (it
// contains __syncthreads); on return with DST_SMEM the results are visible to the whole CTA.
template <typename T, int L, int DIR, bool SRC_SMEM, bool DST_SMEM, class Src, class Dst>
__device__ __forceinline__ void fft_line_io(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws, const Src& src,
                                            const Dst& dst) {
    constexpr int TPL = Tpl<L, T>::V, R = Tpl<L, T>::R;
    if constexpr (L <= R) {
        stage_io<T, L, L, 1, DIR, TPL, SRC_SMEM && DST_SMEM>(t, tw, tws, src, dst);
        if (DST_SMEM) __syncthreads();
    } else {
        stage_io<T, L, R, 1, DIR, TPL, SRC_SMEM>(t, tw, tws, src, SmemLine<T>{buf});
        __syncthreads();
        stages_rest<T, L, DIR, TPL, R, R, DST_SMEM>(buf, t, tw, tws, dst);
    }
}

// in-place line FFT in shared memory
template <typename T, int L, int DIR>
__device__ __forceinline__ void fft_line(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws) {
    fft_line_io<T, L, DIR, true, true>(buf, t, tw, tws, SmemLine<T>{buf}, SmemLine<T>{buf});
}

// ---------------------------------------------------------------------------------------------
// real <-> half-complex post/pre-processing of a row of N = 2L reals packed as L complex
// z_n = x_{2n} + i x_{2n+1}.  After the forward L-point FFT Z, X_k (k = 0..L) of the N-point DFT:
//   E = (Z_k + conj Z_{L-k})/2, O = (Z_k - conj Z_{L-k})/(2i), X_k = E + W^k O, X_{L-k} = conj(E - W^k O),
// W = e^{-2 pi i/N}.  Inverse: Z_k = E + i O with E = (X_k + conj X_{L-k})/2,
// O = (X_k - conj X_{L-k}) conj(W^k)/2, and Z_{L-k} = conj(E) + i conj(O).
template <typename T>
__device__ __forceinline__ void r2c_pair(Cx<T> zk, Cx<T> zl, Cx<T> w, Cx<T>& Xk, Cx<T>& Xl) {
    const Cx<T> E = cx((zk.re + zl.re) * T(0.5), (zk.im - zl.im) * T(0.5));
    const T a = zk.re - zl.re, b = zk.im + zl.im;  // (Z_k - conj Z_{L-k}) / (2i) = (b - ia)/2
    const Cx<T> O = cx(b * T(0.5), -a * T(0.5));
    const Cx<T> WO = cmul(w, O);
    Xk = E + WO;
    Xl = conj(E - WO);
}
template <typename T>
__device__ __forceinline__ void c2r_pair(Cx<T> xk, Cx<T> xl, Cx<T> w, Cx<T>& Zk, Cx<T>& Zl) {
    const Cx<T> E = cx((xk.re + xl.re) * T(0.5), (xk.im - xl.im) * T(0.5));
    const Cx<T> D = cx((xk.re - xl.re) * T(0.5), (xk.im + xl.im) * T(0.5));
    const Cx<T> O = cmul(D, conj(w));
    Zk = cx(E.re - O.im, E.im + O.re);   // E + iO
    Zl = cx(E.re + O.im, -E.im + O.re);  // conj(E) + i conj(O)
}

// Row accessors (row = contiguous line of L complex values)
template <typename Ti, typename Tc>
struct RowLd {  // reads type Ti, widens to Tc
    const Cx<Ti>* p;
    __device__ __forceinline__ Cx<Tc> ld(int i) const {
        const Cx<Ti> v = p[i];
        return cx<Tc>((Tc)v.re, (Tc)v.im);
    }
};
template <typename T>
struct RowSt {  // out = v (+ add) (+ out when acc); nothing when !on
    Cx<T>* p;
    const Cx<T>* add;
    int acc;
    bool on;
    __device__ __forceinline__ void st(int i, const Cx<T>& v) const {
        if (!on) return;
        Cx<T> r = v;
        if (add) r = r + add[i];
        if (acc) r = r + p[i];
        p[i] = r;
    }
};

// Row pass: x1-derivative of real rows ("N2 N3 1D FFTs across the first coordinate,
// diagonal scaling, and then the same number of inverse FFTs").  out = acc*out + d f/dx1.
template <typename T, int L>
struct RowDerivPass {
    using RC = RowCfg<L, T>;
    static constexpr int TPL = RC::TPL, LP = RC::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUF = RC::SMEM;
    Grid g;
    const T* f;
    T* out;
    int accumulate;
    const Cx<T>* twN;
    int64_t cs = 0, cso = 0;  // element strides of f / out between the fields of a batch (blockIdx.y)
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        const T* f = this->f + blockIdx.y * cs;
        T* out = this->out + blockIdx.y * cso;
        const int64_t nrows = (int64_t)g.n2 * g.n3;
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows;
        if (!ok) row = nrows - 1;  // duplicate work on the last row, never stored
        Cx<T>* buf = sm + line * LP;
        const Cx<T>* src = reinterpret_cast<const Cx<T>*>(f) + row * L;
        fft_line_io<T, L, -1, false, true>(buf, t, twN, 2, RowLd<T, T>{src}, SmemLine<T>{buf});
        // post-process pairs (k, L-k), multiply by i k'_1 / L (Nyquist k = L zeroed, reading A2; 1/L
        // normalises the c2r), pre-process back -- all on the same pair, in place
        for (int k = t; k <= L / 2; k += TPL) {
            const int l = (k == 0) ? 0 : L - k;
            Cx<T> Xk, Xl;
            r2c_pair(buf[P(k)], buf[P(l)], twN[k], Xk, Xl);
            // k = 0: Xl is X_L (Nyquist, zeroed); X_0 gets k' = 0
            Xk = mul_i(Xk, T(k) / T(L));
            Xl = (k == 0) ? cx(T(0), T(0)) : mul_i(Xl, T(L - k) / T(L));
            if (k == L / 2 && L > 1) Xl = Xk;  // the same slot (L - k = k)
            Cx<T> Zk, Zl;
            c2r_pair(Xk, (k == 0) ? cx(T(0), T(0)) : Xl, twN[k], Zk, Zl);
            buf[P(k)] = Zk;
            if (k != 0 && 2 * k != L) buf[P(L - k)] = Zl;
        }
        __syncthreads();
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(out) + row * L;
        fft_line_io<T, L, +1, true, false>(buf, t, twN, 2, SmemLine<T>{buf}, RowSt<T>{dst, nullptr, accumulate, ok});
    }
};

// Row pass: real rows (type Ti) -> half-spectrum rows (r2c along x1) computed and stored in Tc,
// spectrum row stride g.n1p.  Ti = float, Tc = double keeps the forward spectrum exact enough for the
// high-wavenumber amplification of beta*A.
template <typename Ti, typename Tc, int L>
struct RowR2cPass {
    using RC = RowCfg<L, Tc>;
    static constexpr int TPL = RC::TPL, LP = RC::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<Tc, NT>::V;
    static constexpr size_t BUF = RC::SMEM;
    Grid g;
    const Ti* f;
    Cx<Tc>* spec;
    const Cx<Tc>* twN;
    int64_t csf = 0, css = 0;  // component strides (blockIdx.y = component) of f and spec
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<Tc>* sm = reinterpret_cast<Cx<Tc>*>(smem);
        const int64_t nrows = (int64_t)g.n2 * g.n3;
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows;
        if (!ok) row = nrows - 1;
        Cx<Tc>* buf = sm + line * LP;
        const Cx<Ti>* src = reinterpret_cast<const Cx<Ti>*>(f + blockIdx.y * csf) + row * L;
        fft_line_io<Tc, L, -1, false, true>(buf, t, twN, 2, RowLd<Ti, Tc>{src}, SmemLine<Tc>{buf});
        if (!ok) return;
        Cx<Tc>* out = spec + blockIdx.y * css + row * g.n1p;
        for (int k = t; k <= L / 2; k += TPL) {
            Cx<Tc> Xk, Xl;
            r2c_pair(buf[P(k)], buf[P(k == 0 ? 0 : L - k)], twN[k], Xk, Xl);
            out[k] = Xk;
            out[L - k] = Xl;  // k = 0 writes X_L; k = L/2 writes the same value twice
        }
    }
};

// Row pass: half-spectrum rows -> real rows (c2r along x1) in T with epilogue out = x + add.
// The spectrum already carries the full inverse normalisation.
template <typename T>
struct RowOut {
    T* out;
    const T* add;  // nullable: field added after the inverse (b~ in the non-isochoric matvec)
};

template <typename T, int L>
struct RowC2rPass {
    using RC = RowCfg<L, T>;
    static constexpr int TPL = RC::TPL, LP = RC::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUF = RC::SMEM;
    Grid g;
    const Cx<T>* spec;
    RowOut<T> epi;
    const Cx<T>* twN;
    int64_t csf = 0, css = 0;  // component strides (blockIdx.y = component) of out/add and spec
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        const int64_t nrows = (int64_t)g.n2 * g.n3;
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows;
        if (!ok) row = nrows - 1;
        Cx<T>* buf = sm + line * LP;
        const Cx<T>* in = spec + blockIdx.y * css + row * g.n1p;
        for (int k = t; k <= L / 2; k += TPL) {
            Cx<T> Zk, Zl;
            c2r_pair(in[k], in[L - k], twN[k], Zk, Zl);
            buf[P(k)] = Zk;
            if (k != 0 && 2 * k != L) buf[P(L - k)] = Zl;
        }
        __syncthreads();
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(epi.out + blockIdx.y * csf) + row * L;
        const Cx<T>* add = epi.add ? reinterpret_cast<const Cx<T>*>(epi.add + blockIdx.y * csf) + row * L : nullptr;
        fft_line_io<T, L, +1, true, false>(buf, t, twN, 2, SmemLine<T>{buf}, RowSt<T>{dst, add, 0, ok});
    }
};

// ---------------------------------------------------------------------------------------------
// Staged row passes (persistent CTAs, bulk-copy prefetch).  x1 rows are contiguous, so a tile of RB
// rows is fetched by the bulk-copy (TMA) engine: warp 0 issues one cp.async.bulk per row into padded
// shared-memory rows and an mbarrier counts the bytes.  Each CTA loops over tiles (tile += gridDim.x)
// with two input stages: tile i+1 is in flight while tile i is transformed, so HBM latency is hidden
// without registers or extra warps.  An epilogue operand (the b~ rows added by the c2r of the matvec)
// is single-buffered: issued at the start of a tile, consumed by its last stage.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!done);
}

// Shared-memory row stride (elements of complex E) of a staged row of n elements read by TPL lanes per
// row: >= n, = TPL (mod W) so the W / TPL rows of one wavefront hit distinct banks, and a multiple of 16
// bytes (bulk-copy destination alignment).
template <typename E, int TPL>
__host__ __device__ constexpr int staged_stride(int n) {
    constexpr int W = WaveLanes<E>::V;
    int v = n;
    if (TPL < W) v = n + (((TPL - n) % W) + W) % W;
    while ((v * (int)sizeof(Cx<E>)) % 16) ++v;  // (only tiny lines: TPL = 1 and an odd stride)
    return v;
}

// Warp 0 (all lanes): fetch rows r0 .. r0 + nr - 1 (bytes per row, global row stride gs bytes) into
// shared rows of stride ss bytes, completing on mbarrier b.
__device__ __forceinline__ void issue_rows(unsigned char* dst, const unsigned char* g, int64_t r0, int nr, int64_t gs,
                                           int ss, unsigned bytes, uint64_t* b, int lane) {
    if (lane == 0) mbar_expect(b, (unsigned)nr * bytes);
    __syncwarp();
    for (int r = lane; r < nr; r += 32) bulk_load(dst + (size_t)r * ss, g + (r0 + r) * gs, bytes, b);
}

template <int L, typename Tc>
struct StagedRowCfg {
    static constexpr int TPL = Tpl<L, Tc>::V;
    static constexpr int NT = 128;
    static constexpr int RB = NT / TPL;
    static constexpr int LP = RowLP<L, Tc, TPL>::V;
    static constexpr size_t LINES = (size_t)RB * LP * sizeof(Cx<Tc>);
};

// r2c along x1 (as RowR2cPass) from staged rows of Ti.
template <typename Ti, typename Tc, int L>
struct RowR2cStaged {
    using RC = StagedRowCfg<L, Tc>;
    static constexpr int TPL = RC::TPL, LP = RC::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<Tc, NT>::V;
    static constexpr int SI = staged_stride<Ti, TPL>(L) * (int)sizeof(Cx<Ti>);  // staged row stride, bytes
    static constexpr size_t STG = (size_t)RB * SI, EPB = 0;
    static constexpr int NTW = 2 * L;  // twiddles e^{-2 pi i m / 2L} in shared memory
    static constexpr int NST = stage_tw_count<L, 16>();  // + the stage-major table of the L-point FFT
    using TW = Cx<Tc>;
    static constexpr size_t BUF = 128 + 2 * STG + EPB + RC::LINES + (NTW + NST) * sizeof(TW);
    Grid g;
    const Ti* f;
    Cx<Tc>* spec;
    const Cx<Tc>* twN;
    int64_t csf = 0, css = 0;  // component strides (blockIdx.y = component)
    __device__ __forceinline__ int64_t nrows() const { return (int64_t)g.n2 * g.n3; }
    __device__ __forceinline__ void issue_in(int tile, unsigned char* dst, uint64_t* b, int lane) const {
        const int64_t r0 = (int64_t)tile * RB;
        const int nr = (int)min((int64_t)RB, nrows() - r0);
        issue_rows(dst, reinterpret_cast<const unsigned char*>(f + blockIdx.y * csf), r0, nr,
                   (int64_t)L * sizeof(Cx<Ti>), SI, L * sizeof(Cx<Ti>), b, lane);
    }
    __device__ __forceinline__ void issue_ep(int, unsigned char*, uint64_t*, int) const {}
    __device__ __forceinline__ void run(int tile, const unsigned char* stg, const unsigned char*, uint64_t*, unsigned,
                                        unsigned char* lines, const TW* twN) const {
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        const int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows();
        Cx<Tc>* buf = reinterpret_cast<Cx<Tc>*>(lines) + line * LP;
        const Cx<Ti>* src = reinterpret_cast<const Cx<Ti>*>(stg + line * SI);
        fft_line_io<Tc, L, -1, false, true>(buf, t, twN + NTW, -1, RowLd<Ti, Tc>{src}, SmemLine<Tc>{buf});
        if (!ok) return;
        Cx<Tc>* out = spec + blockIdx.y * css + row * g.n1p;
        for (int k = t; k <= L / 2; k += TPL) {
            Cx<Tc> Xk, Xl;
            r2c_pair(buf[P(k)], buf[P(k == 0 ? 0 : L - k)], twN[k], Xk, Xl);
            out[k] = Xk;
            out[L - k] = Xl;
        }
    }
};

// c2r along x1 (as RowC2rPass) from staged spectrum rows; ADD: + staged real rows of epi.add.
template <typename T, int L, bool ADD>
struct RowC2rStaged {
    using RC = StagedRowCfg<L, T>;
    static constexpr int TPL = RC::TPL, LP = RC::LP, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr int NIN = L + 2;  // complex values fetched per spectrum row (L + 1 used; 16-byte multiple)
    static constexpr int SI = staged_stride<T, TPL>(NIN) * (int)sizeof(Cx<T>);
    static constexpr int SA = staged_stride<T, TPL>(L) * (int)sizeof(Cx<T>);
    static constexpr size_t STG = (size_t)RB * SI, EPB = ADD ? (size_t)RB * SA : 0;
    static constexpr int NTW = 2 * L;
    static constexpr int NST = stage_tw_count<L, 16>();
    using TW = Cx<T>;
    static constexpr size_t BUF = 128 + 2 * STG + EPB + RC::LINES + (NTW + NST) * sizeof(TW);
    Grid g;
    const Cx<T>* spec;
    RowOut<T> epi;
    const Cx<T>* twN;
    int64_t csf = 0, css = 0;  // component strides (blockIdx.y = component) of out/add and spec
    __device__ __forceinline__ int64_t nrows() const { return (int64_t)g.n2 * g.n3; }
    __device__ __forceinline__ void issue_in(int tile, unsigned char* dst, uint64_t* b, int lane) const {
        const int64_t r0 = (int64_t)tile * RB;
        const int nr = (int)min((int64_t)RB, nrows() - r0);
        issue_rows(dst, reinterpret_cast<const unsigned char*>(spec + blockIdx.y * css), r0, nr,
                   (int64_t)g.n1p * sizeof(Cx<T>), SI, NIN * sizeof(Cx<T>), b, lane);
    }
    __device__ __forceinline__ void issue_ep(int tile, unsigned char* dst, uint64_t* b, int lane) const {
        if constexpr (ADD) {
            const int64_t r0 = (int64_t)tile * RB;
            const int nr = (int)min((int64_t)RB, nrows() - r0);
            issue_rows(dst, reinterpret_cast<const unsigned char*>(epi.add + blockIdx.y * csf), r0, nr,
                       (int64_t)L * sizeof(Cx<T>), SA, L * sizeof(Cx<T>), b, lane);
        }
    }
    __device__ __forceinline__ void run(int tile, const unsigned char* stg, const unsigned char* ep, uint64_t* epb,
                                        unsigned epar, unsigned char* lines, const TW* twN) const {
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        const int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows();
        Cx<T>* buf = reinterpret_cast<Cx<T>*>(lines) + line * LP;
        const Cx<T>* in = reinterpret_cast<const Cx<T>*>(stg + line * SI);
        for (int k = t; k <= L / 2; k += TPL) {
            Cx<T> Zk, Zl;
            c2r_pair(in[k], in[L - k], twN[k], Zk, Zl);
            buf[P(k)] = Zk;
            if (k != 0 && 2 * k != L) buf[P(L - k)] = Zl;
        }
        __syncthreads();
        const Cx<T>* add = nullptr;
        if constexpr (ADD) {
            mbar_wait(epb, epar);
            add = reinterpret_cast<const Cx<T>*>(ep + line * SA);
        }
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(epi.out + blockIdx.y * csf) + row * L;
        fft_line_io<T, L, +1, true, false>(buf, t, twN + NTW, -1, SmemLine<T>{buf}, RowSt<T>{dst, add, 0, ok});
    }
};

// Persistent driver of a staged row pass: grid = min(tiles, resident CTAs); barriers 0/1 = input stages,
// 2 = epilogue operand.
template <class PassT>
__global__ void __launch_bounds__(PassT::NT, PassT::MINB) k_rows(PassT pass, int ntiles) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* stg = smem_raw + 128;
    unsigned char* ep = stg + 2 * PassT::STG;
    unsigned char* lines = ep + PassT::EPB;
    // the pass's twiddle table, read by every butterfly: copied once per CTA (in L1 it would be evicted
    // by the streaming traffic and every miss stalls a dependent multiply on an L2 round trip)
    typename PassT::TW* tw = reinterpret_cast<typename PassT::TW*>(lines + PassT::RC::LINES);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 1);
        mbar_fence_init();
    }
    for (int i = threadIdx.x; i < PassT::NTW; i += PassT::NT) tw[i] = pass.twN[i];
    // stage-major table (stage_tw_off): entry (Ns, r, k) = twN[2 r k L / (Ns Rs)] of the L-point plan
    constexpr int L = PassT::NTW / 2;
    for (int i = threadIdx.x; i < PassT::NST; i += PassT::NT) {
        int Ns = 16, e = i;
        while (e >= ((L / Ns < 16 ? L / Ns : 16) - 1) * Ns) {
            e -= ((L / Ns < 16 ? L / Ns : 16) - 1) * Ns;
            Ns *= 16;
        }
        const int Rs = L / Ns < 16 ? L / Ns : 16;
        const int r = 1 + e / Ns, k = e % Ns;
        tw[PassT::NTW + i] = pass.twN[2 * r * k * (L / (Ns * Rs))];
    }
    __syncthreads();
    int tile = blockIdx.x;
    if (warp == 0 && tile < ntiles) pass.issue_in(tile, stg, &bar[0], lane);
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const int st = it & 1;
        if (warp == 0) {
            // the other stage and the epilogue buffer were last read before the previous trailing barrier
            if (tile + (int)gridDim.x < ntiles) pass.issue_in(tile + gridDim.x, stg + (st ^ 1) * PassT::STG, &bar[st ^ 1], lane);
            if (PassT::EPB) pass.issue_ep(tile, ep, &bar[2], lane);
        }
        mbar_wait(&bar[st], (unsigned)(it >> 1) & 1u);
        pass.run(tile, stg + st * PassT::STG, ep, &bar[2], (unsigned)it & 1u, lines, tw);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// Column passes along x2 (AX = 2) or x3 (AX = 3) of a complex array with W complex columns per row
// (W = n1p for spectra, N1/2 for a real field read as pairs) and extents (W, n2, n3).
// A CTA owns XC consecutive columns x OL lines of the other transverse axis; consecutive lanes own
// consecutive columns, so every global access of a stage is a full 128-byte segment.
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

// Element p of one line of a column array: address base + p * lo in the plain layouts, base +
// (p >> sh) * hi + (p & mk) * lo in the split layout (blocks of nb = 2^sh lines).  SPLIT is a template
// flag so the single-GPU passes carry no 64-bit block arithmetic (the plain offset p * lo < 2^31:
// lo <= n2 * n1p and p < n3 for every supported grid).
// Out-of-range lines (on = false) read 0 and store nothing.
template <typename T, bool SPLIT = false>
struct ColAcc {
    Cx<T>* b;
    int64_t hi;
    int lo, sh, mk;
    bool on;
    int acc;
    __device__ __forceinline__ int64_t at(int p) const {
        if constexpr (SPLIT) return (int64_t)(p >> sh) * hi + (int64_t)(p & mk) * lo;
        else return p * lo;
    }
    __device__ __forceinline__ Cx<T> ld(int p) const { return on ? b[at(p)] : cx(T(0), T(0)); }
    __device__ __forceinline__ void st(int p, const Cx<T>& v) const {
        if (!on) return;
        Cx<T>* q = b + at(p);
        *q = acc ? v + *q : v;
    }
};

template <int AX, typename T, bool SPLIT = false>
__device__ __forceinline__ ColAcc<T, SPLIT> col_acc(Cx<T>* a, const ColGeom& c, int x, int o, int nb, bool on, int acc) {
    ColAcc<T, SPLIT> r;
    r.on = on;
    r.acc = acc;
    r.sh = 30;
    r.mk = 0x3fffffff;
    r.hi = 0;
    if (!on) {
        x = 0;
        o = 0;
    }
    if (AX == 2) {
        r.lo = c.W;
        if (nb) {
            int l = 0;
            while ((1 << l) < nb) ++l;
            r.sh = l;
            r.mk = nb - 1;
            r.hi = (int64_t)c.n3 * nb * c.W;
            r.b = a + ((int64_t)o * nb) * c.W + x;
        } else {
            r.b = a + ((int64_t)o * c.n2) * c.W + x;
        }
    } else {
        r.lo = c.n2 * c.W;
        r.b = a + (int64_t)o * c.W + x;
    }
    return r;
}

// Fused all-to-all transposes (multi-GPU x3 slabs, SURVEY §8(e) "FFT pass epilogues ... store straight
// into peer buffers"): the last stage of the pass that produces a transpose's send data stores each
// element straight into the receive buffer of the rank that owns it (peer memory), in the layout the
// all-to-all would have delivered.  pws[q]: rank q's workspace as mapped here (a device array), boff:
// byte offset of the receive buffer plus this rank's chunk.  Element p of the line goes to rank
// q = p >> sh at pws[q] + boff + (ofs + (p & mk) * lo) elements.
template <typename T>
struct PeerAcc {
    char* const* pws;
    int64_t boff, ofs;
    int64_t lo;
    int sh, mk;
    bool on;
    __device__ __forceinline__ void st(int p, const Cx<T>& v) const {
        if (!on) return;
        reinterpret_cast<Cx<T>*>(pws[p >> sh] + boff)[ofs + (int64_t)(p & mk) * lo] = v;
    }
};
struct PeerDst {  // host-filled description of a peer destination (nullptr pws: plain stores)
    char* const* pws = nullptr;
    int64_t boff = 0;
    int sh = 0;
};
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

// CTA shape of a column pass: XC columns (one 128-byte segment: 16 complex64 / 8 complex128) x OL
// transverse lines, TPL threads per line, capped so NC components of the CTA's lines fit in ~96 KB.
// MAXNT > 0 caps the CTA at MAXNT threads by narrowing XC (the fp64 x3 middle pass at L >= 512: 32
// threads per line x 8 columns made 256-thread CTAs of ~200 registers, one per SM -- 8 warps, latency
// bound at 2 TB/s; 4 columns x 32 threads keep 2-3 CTAs per SM).
template <int L, typename T, int NC = 1, int MAXNT = 0>
struct ColCfg {
    static constexpr int ES = (int)sizeof(Cx<T>);
    static constexpr int TPL = Tpl<L, T>::V;
    static constexpr int LPB = (L + L / 16 + 1 + WaveLanes<T>::V) * ES;  // bytes per line (bound, for sizing)
    static constexpr int XCN = (MAXNT > 0 && MAXNT / TPL >= 1 && MAXNT / TPL < 128 / ES) ? MAXNT / TPL : 128 / ES;
    static constexpr int XC0 = XCN;
    static constexpr int XC = (NC * XC0 * LPB <= 96 * 1024) ? XC0 : (NC * (XC0 / 2) * LPB <= 96 * 1024) ? (XC0 / 2 > 0 ? XC0 / 2 : 1) : (XC0 / 4 > 0 ? XC0 / 4 : 1);
    static constexpr int OLT = (XC * TPL >= CtaThreads<T>::V) ? 1 : CtaThreads<T>::V / (XC * TPL);
    static constexpr int MAXL = (96 * 1024) / (NC * LPB);
    static constexpr int OLS = (MAXL / XC) >= 1 ? MAXL / XC : 1;
    static constexpr int OL = OLT < OLS ? OLT : OLS;
    static constexpr int NT = XC * OL * TPL;
    static constexpr int LINES = XC * OL;
    static constexpr int LP = ColLP<L, T, XC>::V;
    static constexpr size_t SMEM = (size_t)NC * LINES * LP * ES;
};

// Twiddle table of a column pass copied into shared memory at the start of the CTA (an L1-resident
// table is evicted by the streaming traffic, and every miss stalls a dependent multiply on L2).  Only
// stages with Ns > 1 read twiddles, and the first stage of every line is followed by a barrier, so
// the copy needs no barrier of its own.  Measured at 256^3: fp32 passes 4-7 % faster; the fp64 middle
// pass 8 % slower (its 16-byte twiddle reads conflict in shared memory), so fp64 passes keep L1.
template <typename T, int L, int NT, bool ON>
__device__ __forceinline__ const Cx<T>* tw_smem(const Cx<T>* __restrict__ tw, Cx<T>* sm) {
    if constexpr (!ON) return tw;
    for (int i = threadIdx.x; i < L; i += NT) sm[i] = tw[i];
    return sm;
}

// CTA-size cap of the fp32 derivative / x2 column passes at L >= 512 (16 columns x 32 threads made
// 512-thread CTAs, one or two per SM; 8 columns: the x3 derivative 1.38 -> 0.92 ms, the inverse x2 pass
// 854 -> 697 us at 512^3; the fp64 x2 pass measured slower capped, 1200 -> 1375 us, and is not)
template <int L, typename T>
struct ColCap {
    static constexpr int V = (L >= 512 && sizeof(T) == 4) ? CtaThreads<T>::V : 0;
};

// thread -> (column xi, thread-in-line t, transverse line oi); line index oi * XC + xi
template <int XC, int TPL>
__device__ __forceinline__ void col_thread(int& xi, int& t, int& oi) {
    xi = threadIdx.x % XC;
    const int r = threadIdx.x / XC;
    t = r % TPL;
    oi = r / TPL;
}

template <int XC, int OL>
__device__ __forceinline__ void col_origin(const ColGeom& c, int tile, int& x0, int& o0) {
    const int nxb = (c.nx + XC - 1) / XC;
    x0 = (tile % nxb) * XC;
    o0 = (tile / nxb) * OL;
}

// Derivative along x2 / x3 of a real field (viewed as complex pairs): out (+)= d f / dx_AX.
template <typename T, int L, int AX>
struct ColDerivPass {
    using CC = ColCfg<L, T, 1, ColCap<L, T>::V>;
    static constexpr int TPL = CC::TPL, LP = CC::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr bool TWS = sizeof(T) == 4;
    static constexpr size_t BUF = CC::SMEM + (TWS ? L * sizeof(Cx<T>) : 0);  // + twiddles
    ColGeom c;
    const Cx<T>* src;
    Cx<T>* dst;
    int accumulate;
    const Cx<T>* tw;
    int64_t cs = 0, cso = 0;  // complex-element strides of src / dst between the fields of a batch (blockIdx.y)
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        const Cx<T>* src = this->src + blockIdx.y * cs;
        Cx<T>* dst = this->dst + blockIdx.y * cso;
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int x = x0 + xi, o = o0 + oi, nother = (AX == 2) ? c.n3 : c.n2;
        const bool on = x < c.nx && o < nother;
        Cx<T>* buf = sm + (oi * XC + xi) * LP;
        const Cx<T>* tw = tw_smem<T, L, NT, TWS>(this->tw, reinterpret_cast<Cx<T>*>(smem + CC::SMEM));
        fft_line_io<T, L, -1, false, true>(buf, t, tw, 1, col_acc<AX>(const_cast<Cx<T>*>(src), c, x, o, 0, on, 0),
                                           SmemLine<T>{buf});
        for (int k = t; k < L; k += TPL) {
            const T kp = (T)wavenum_odd(k, L);
            buf[P(k)] = mul_i(buf[P(k)], kp / T(L));
        }
        __syncthreads();
        fft_line_io<T, L, +1, true, false>(buf, t, tw, 1, SmemLine<T>{buf}, col_acc<AX>(dst, c, x, o, 0, on, accumulate));
    }
};

// Complex FFT of spectrum columns along x2 (forward DIR=-1 or inverse DIR=+1), src -> dst (may alias
// when both layouts are plain: every element is read by its own CTA before that CTA writes it).
// nb_in / nb_out != 0 select the split layout on that side (the all-to-all chunks of the multi-GPU
// transposes), fusing the pack / unpack into this pass.
// DCS: dst has its own component stride csd (the scratch ring); a template flag because the runtime
// choice cost the plain passes 8 % (fp32 x2: 83 -> 90 us at 256^3)
template <typename T, int L, int DIR, bool SPLIT_IN = false, bool SPLIT_OUT = false, bool PEER = false, bool DCS = false>
struct ColFftPass {
    using CC = ColCfg<L, T, 1, ColCap<L, T>::V>;
    static constexpr int TPL = CC::TPL, LP = CC::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr bool TWS = sizeof(T) == 4;
    static constexpr size_t BUF = CC::SMEM + (TWS ? L * sizeof(Cx<T>) : 0);  // + twiddles
    ColGeom c;
    const Cx<T>* src;
    Cx<T>* dst;
    const Cx<T>* tw;
    int nb_in, nb_out;
    int64_t cs = 0;    // component stride (blockIdx.y = component) of src (and of dst when csd < 0)
    int64_t csd = -1;  // component stride of dst
    PeerDst pd;        // PEER: the split-layout chunks go straight to their ranks' receive buffers
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int x = x0 + xi, o = o0 + oi;
        const bool on = x < c.nx && o < c.n3;
        Cx<T>* buf = sm + (oi * XC + xi) * LP;
        const Cx<T>* tw = tw_smem<T, L, NT, TWS>(this->tw, reinterpret_cast<Cx<T>*>(smem + CC::SMEM));
        if constexpr (PEER) {  // chunk of rank q = x2 block q: [i3][i2 % nb][x] in q's receive buffer
            const int nb = nb_out;
            PeerAcc<T> pa{pd.pws, pd.boff, ((int64_t)o * nb) * c.W + x, c.W, pd.sh, nb - 1, on};
            fft_line_io<T, L, DIR, false, false>(
                buf, t, tw, 1, col_acc<2, T, SPLIT_IN>(const_cast<Cx<T>*>(src) + blockIdx.y * cs, c, x, o, nb_in, on, 0), pa);
            return;
        }
        fft_line_io<T, L, DIR, false, false>(buf, t, tw, 1,
                                             col_acc<2, T, SPLIT_IN>(const_cast<Cx<T>*>(src) + blockIdx.y * cs, c, x, o, nb_in, on, 0),
                                             col_acc<2, T, SPLIT_OUT>(dst + blockIdx.y * (DCS ? csd : cs), c, x, o, nb_out, on, 0));
    }
};

// Isochoric data term, x2 stage (L b~ = b~ - grad Lap^-1 div b~, Eq. 4): from the x1 half
// spectra P_a = F1 b~_a of the three components it forms Q = i (k1' F2 P_1 + k2' F2 P_2) and R = F2 P_3,
// so that the x3 middle pass obtains F[div b~] = F3 Q + i k3' F3 R (the spectral divergence with the
// Nyquist wavenumbers zeroed, as the derivative passes take it) -- no real-space derivative passes and
// no forward transform of div b~.  Q may alias P_1 and R alias P_3 in the plain layout (every element is
// read by its own CTA before that CTA writes it); SPLIT_OUT writes the all-to-all split layout (slabs).
template <typename T, int L, bool SPLIT_OUT = false>
struct ColDivPass {
    using CC = ColCfg<L, T, 2, ColCap<L, T>::V>;
    static constexpr int TPL = CC::TPL, LP = CC::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT, LINES = CC::LINES;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr bool TWS = sizeof(T) == 4;
    static constexpr size_t BUF = CC::SMEM + (TWS ? L * sizeof(Cx<T>) : 0);  // + twiddles
    ColGeom c;
    const Cx<T>* p1;
    const Cx<T>* p2;
    const Cx<T>* p3;
    Cx<T>* q;
    Cx<T>* r;
    const Cx<T>* tw;
    int nb_out;
    int n1;  // real x1 extent: column n1 / 2 is the x1 Nyquist
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int x = x0 + xi, o = o0 + oi;
        const bool on = x < c.nx && o < c.n3;
        Cx<T>* bA = sm + (oi * XC + xi) * LP;
        Cx<T>* bB = bA + LINES * LP;
        const Cx<T>* tw = tw_smem<T, L, NT, TWS>(this->tw, reinterpret_cast<Cx<T>*>(smem + CC::SMEM));
        fft_line_io<T, L, -1, false, true>(bA, t, tw, 1, col_acc<2>(const_cast<Cx<T>*>(p1), c, x, o, 0, on, 0),
                                           SmemLine<T>{bA});
        fft_line_io<T, L, -1, false, true>(bB, t, tw, 1, col_acc<2>(const_cast<Cx<T>*>(p2), c, x, o, 0, on, 0),
                                           SmemLine<T>{bB});
        const T k1 = (T)((x == n1 / 2) ? 0 : x);
        const auto qa = col_acc<2, T, SPLIT_OUT>(q, c, x, o, nb_out, on, 0);
        for (int p = t; p < L; p += TPL) {
            const T k2 = (T)wavenum_odd(p, L);
            qa.st(p, mul_i(scale(bA[P(p)], k1) + scale(bB[P(p)], k2), T(1)));
        }
        __syncthreads();  // bA is the next transform's line buffer
        fft_line_io<T, L, -1, false, false>(bA, t, tw, 1, col_acc<2>(const_cast<Cx<T>*>(p3), c, x, o, 0, on, 0),
                                            col_acc<2, T, SPLIT_OUT>(r, c, x, o, nb_out, on, 0));
    }
};

// ---------------------------------------------------------------------------------------------
// x2 lines of a length N that is not a power of two (the paper's 256 x 300 x 256 grid; SURVEY
// §8(b) admits any even N >= 4): Bluestein's chirp-z form of the length-N DFT, X_k = w_k sum_n (x_n w_n)
// conj(w_{k-n}) with w_j = e^{DIR i pi j^2 / N} (nk = (n^2 + k^2 - (k - n)^2) / 2), i.e. a circular
// convolution evaluated with two radix-16 FFTs of the power of two M >= 2N - 1 and the precomputed
// transform bhat = FFT_M(b) / M of the chirp b_j = conj(w_j), j in (-N, N).  chirp[n] = w_n per direction.
// Plain x2 transforms compute in their I/O precision (the forward of the amplifying symbols is fp64 by
// type, reading A20; an fp32 inverse after a symbol rounds relative to the already-shaped signal); the
// derivative and divergence stages compute in fp64 whatever the I/O type: an fp32 convolution of length
// M ~ 2N leaves a white rounding floor that the odd symbol (k' / N up to N / 2) lifts past the 1e-5
// operator bar.
template <typename Ti, typename Tc>
struct AccC {  // a column accessor in the I/O type, seen in the compute type
    ColAcc<Ti> a;
    __device__ __forceinline__ Cx<Tc> ld(int i) const {
        const Cx<Ti> v = a.ld(i);
        return cx<Tc>((Tc)v.re, (Tc)v.im);
    }
    __device__ __forceinline__ void st(int i, const Cx<Tc>& v) const { a.st(i, cx<Ti>((Ti)v.re, (Ti)v.im)); }
};
template <typename Ti>
using AccD = AccC<Ti, double>;
template <typename Tc, class Src>
struct ChirpLd {  // a_j = w_j x_j (j < n), zero padding up to M
    Src s;
    const Cx<Tc>* w;
    int n;
    __device__ __forceinline__ Cx<Tc> ld(int j) const { return j < n ? cmul(s.ld(j), w[j]) : cx(Tc(0), Tc(0)); }
};
template <typename Tc, class Dst>
struct ChirpSt {  // X_k = w_k c_k (k < n); the padding outputs are dropped
    Dst d;
    const Cx<Tc>* w;
    int n;
    __device__ __forceinline__ void st(int k, const Cx<Tc>& v) const {
        if (k < n) d.st(k, cmul(v, w[k]));
    }
};
template <typename Tc>
struct BlueTab {  // twM[M], then for the forward (0) / inverse (1) direction w[N], bhat[M]
    const Cx<Tc>* twM;
    const Cx<Tc>* w[2];
    const Cx<Tc>* bhat[2];
    int n;
};
template <typename Tc, int M, int D, class Src, class Dst>
__device__ __forceinline__ void blue_line(Cx<Tc>* buf, int t, const BlueTab<Tc>& bt, const Src& src, const Dst& dst) {
    constexpr int TPL = Tpl<M, Tc>::V;
    fft_line_io<Tc, M, -1, false, true>(buf, t, bt.twM, 1, ChirpLd<Tc, Src>{src, bt.w[D], bt.n}, SmemLine<Tc>{buf});
    for (int j = t; j < M; j += TPL) buf[P(j)] = cmul(buf[P(j)], bt.bhat[D][j]);
    __syncthreads();
    fft_line_io<Tc, M, +1, true, false>(buf, t, bt.twM, 1, SmemLine<Tc>{buf}, ChirpSt<Tc, Dst>{dst, bt.w[D], bt.n});
}

// x2 FFT (DIR) of length N = bt.n in T, src -> dst (may alias: a CTA loads its lines before it stores them)
template <typename T, int M, int DIR>
struct ColBlueFftPass {
    using CC = ColCfg<M, T, 1, ColCap<M, T>::V>;
    static constexpr int TPL = CC::TPL, LP = CC::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT;
    static constexpr int MINB = MinB<T, NT>::V;
    static constexpr size_t BUF = CC::SMEM;
    ColGeom c;
    const Cx<T>* src;
    Cx<T>* dst;
    BlueTab<T> bt;
    int64_t cs = 0, csd = -1;
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int x = x0 + xi, o = o0 + oi;
        const bool on = x < c.nx && o < c.n3;
        blue_line<T, M, DIR < 0 ? 0 : 1>(reinterpret_cast<Cx<T>*>(smem) + (oi * XC + xi) * LP, t, bt,
                                         col_acc<2>(const_cast<Cx<T>*>(src) + blockIdx.y * cs, c, x, o, 0, on, 0),
                                         col_acc<2>(dst + blockIdx.y * (csd >= 0 ? csd : cs), c, x, o, 0, on, 0));
    }
};

// x1 rows of an extent N1 = 2L that is not a power of two (one rank, N1 % 4 == 0): the half-length
// complex transform of the packed row (z_n = x_2n + i x_2n+1, r2c_pair / c2r_pair as the radix passes)
// runs in Bluestein form with M >= 2L - 1.  RB rows per CTA, one M-point work line and one L-point line
// each; every row is processed by TPL = Tpl<M, Tc> threads.
template <int M, typename Tc>
struct RowBlueCfg {
    static constexpr int TPL = Tpl<M, Tc>::V;
    static constexpr int RB = (128 / TPL) > 0 ? 128 / TPL : 1;
    static constexpr int NT = RB * TPL;
    static constexpr int LW = PadLP<M, 1, 0>::V;          // work line
    static constexpr int LZ = M / 2 + M / 32 + 2;           // L <= M / 2 points, padded by P()
    static constexpr size_t SMEM = (size_t)RB * (LW + LZ) * sizeof(Cx<Tc>);
};
template <typename Ti, typename Tc>
struct RowStC {  // a RowSt in the I/O type fed in the compute type
    RowSt<Ti> r;
    __device__ __forceinline__ void st(int i, const Cx<Tc>& v) const { r.st(i, cx<Ti>((Ti)v.re, (Ti)v.im)); }
};
// r2c: real rows (Ti) -> half spectra (Tc), row stride g.n1p
template <typename Ti, typename Tc, int M>
struct RowBlueR2cPass {
    using RC = RowBlueCfg<M, Tc>;
    static constexpr int TPL = RC::TPL, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = 1;
    static constexpr size_t BUF = RC::SMEM;
    Grid g;
    const Ti* f;
    Cx<Tc>* spec;
    const Cx<Tc>* twN;  // e^{-2 pi i m / N1}
    BlueTab<Tc> bt;     // length L = N1 / 2
    int64_t csf = 0, css = 0;
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        const int L = bt.n;
        const int64_t nrows = (int64_t)g.n2 * g.n3;
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows;
        if (!ok) row = nrows - 1;
        Cx<Tc>* work = reinterpret_cast<Cx<Tc>*>(smem) + line * RC::LW;
        Cx<Tc>* z = reinterpret_cast<Cx<Tc>*>(smem) + RB * RC::LW + line * RC::LZ;
        const Cx<Ti>* src = reinterpret_cast<const Cx<Ti>*>(f + blockIdx.y * csf) + row * L;
        blue_line<Tc, M, 0>(work, t, bt, RowLd<Ti, Tc>{src}, SmemLine<Tc>{z});
        __syncthreads();
        if (!ok) return;
        Cx<Tc>* out = spec + blockIdx.y * css + row * g.n1p;
        for (int k = t; k <= L / 2; k += TPL) {
            Cx<Tc> Xk, Xl;
            r2c_pair(z[P(k)], z[P(k == 0 ? 0 : L - k)], twN[k], Xk, Xl);
            out[k] = Xk;
            out[L - k] = Xl;
        }
    }
};
// c2r: half spectra -> real rows (+ add), in T
template <typename T, int M>
struct RowBlueC2rPass {
    using RC = RowBlueCfg<M, T>;
    static constexpr int TPL = RC::TPL, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = 1;
    static constexpr size_t BUF = RC::SMEM;
    Grid g;
    const Cx<T>* spec;
    RowOut<T> epi;
    const Cx<T>* twN;
    BlueTab<T> bt;
    int64_t csf = 0, css = 0;
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        const int L = bt.n;
        const int64_t nrows = (int64_t)g.n2 * g.n3;
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows;
        if (!ok) row = nrows - 1;
        Cx<T>* work = reinterpret_cast<Cx<T>*>(smem) + line * RC::LW;
        Cx<T>* z = reinterpret_cast<Cx<T>*>(smem) + RB * RC::LW + line * RC::LZ;
        const Cx<T>* in = spec + blockIdx.y * css + row * g.n1p;
        for (int k = t; k <= L / 2; k += TPL) {
            Cx<T> Zk, Zl;
            c2r_pair(in[k], in[L - k], twN[k], Zk, Zl);
            z[P(k)] = Zk;
            if (k != 0 && 2 * k != L) z[P(L - k)] = Zl;
        }
        __syncthreads();
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(epi.out + blockIdx.y * csf) + row * L;
        const Cx<T>* add = epi.add ? reinterpret_cast<const Cx<T>*>(epi.add + blockIdx.y * csf) + row * L : nullptr;
        blue_line<T, M, 1>(work, t, bt, SmemLine<T>{z}, RowSt<T>{dst, add, 0, ok});
    }
};
// x1 derivative (RowDerivPass with Bluestein transforms, fp64 arithmetic: the odd symbol lifts an fp32
// convolution's rounding floor), out = acc * out + d f / dx1; nf fields per launch (blockIdx.y)
template <typename T, int M>
struct RowBlueDerivPass {
    using RC = RowBlueCfg<M, double>;
    static constexpr int TPL = RC::TPL, RB = RC::RB, NT = RC::NT;
    static constexpr int MINB = 1;
    static constexpr size_t BUF = RC::SMEM;
    Grid g;
    const T* f;
    T* out;
    int accumulate;
    const Cx<double>* twN;
    BlueTab<double> bt;
    int64_t cs = 0, cso = 0;
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        const int L = bt.n;
        const int64_t nrows = (int64_t)g.n2 * g.n3;
        const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
        int64_t row = (int64_t)tile * RB + line;
        const bool ok = row < nrows;
        if (!ok) row = nrows - 1;
        Cx<double>* work = reinterpret_cast<Cx<double>*>(smem) + line * RC::LW;
        Cx<double>* z = reinterpret_cast<Cx<double>*>(smem) + RB * RC::LW + line * RC::LZ;
        const Cx<T>* src = reinterpret_cast<const Cx<T>*>(f + blockIdx.y * cs) + row * L;
        blue_line<double, M, 0>(work, t, bt, RowLd<T, double>{src}, SmemLine<double>{z});
        __syncthreads();
        for (int k = t; k <= L / 2; k += TPL) {  // RowDerivPass's pair arithmetic
            const int l = (k == 0) ? 0 : L - k;
            Cx<double> Xk, Xl;
            r2c_pair(z[P(k)], z[P(l)], twN[k], Xk, Xl);
            Xk = mul_i(Xk, double(k) / double(L));
            Xl = (k == 0) ? cx(0.0, 0.0) : mul_i(Xl, double(L - k) / double(L));
            if (k == L / 2 && L > 1 && 2 * k == L) Xl = Xk;
            Cx<double> Zk, Zl;
            c2r_pair(Xk, (k == 0) ? cx(0.0, 0.0) : Xl, twN[k], Zk, Zl);
            z[P(k)] = Zk;
            if (k != 0 && 2 * k != L) z[P(L - k)] = Zl;
        }
        __syncthreads();
        Cx<T>* dst = reinterpret_cast<Cx<T>*>(out + blockIdx.y * cso) + row * L;
        blue_line<double, M, 1>(work, t, bt, SmemLine<double>{z}, RowStC<T, double>{RowSt<T>{dst, nullptr, accumulate, ok}});
    }
};

// x2 derivative of a real field viewed as complex pairs (ColDerivPass with Bluestein transforms):
// out (+)= F2^-1[i k2' / N F2 f]; nf fields per launch (blockIdx.y)
template <typename Ti, int M, int AX = 2>
struct ColBlueDerivPass {
    using CC = ColCfg<M, double, 2>;
    static constexpr int TPL = CC::TPL, LP = CC::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT, LINES = CC::LINES;
    static constexpr int MINB = MinB<double, NT>::V;
    static constexpr size_t BUF = CC::SMEM;
    ColGeom c;
    const Cx<Ti>* src;
    Cx<Ti>* dst;
    int accumulate;
    BlueTab<double> bt;
    int64_t cs = 0, cso = 0;
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int x = x0 + xi, o = o0 + oi;
        const bool on = x < c.nx && o < (AX == 2 ? c.n3 : c.n2);
        Cx<double>* bA = reinterpret_cast<Cx<double>*>(smem) + (oi * XC + xi) * LP;
        Cx<double>* bB = bA + LINES * LP;
        const int n = bt.n;
        blue_line<double, M, 0>(bA, t, bt, AccD<Ti>{col_acc<AX>(const_cast<Cx<Ti>*>(src) + blockIdx.y * cs, c, x, o, 0, on, 0)},
                        SmemLine<double>{bB});
        __syncthreads();
        for (int k = t; k < n; k += TPL) bB[P(k)] = mul_i(bB[P(k)], (double)wavenum_odd(k, n) / (double)n);
        __syncthreads();
        blue_line<double, M, 1>(bA, t, bt, SmemLine<double>{bB}, AccD<Ti>{col_acc<AX>(dst + blockIdx.y * cso, c, x, o, 0, on, accumulate)});
    }
};

// ColDivPass with Bluestein x2 transforms: Q = i (k1' F2 P1 + k2' F2 P2), R = F2 P3 (one rank)
template <typename Ti>
struct DivCombineSt {  // Q_k = i (k1' B_k + k2'(k) v)
    Cx<double>* b;
    AccD<Ti> q;
    double k1;
    int n;
    __device__ __forceinline__ void st(int k, const Cx<double>& v) const {
        q.st(k, mul_i(scale(b[P(k)], k1) + scale(v, (double)wavenum_odd(k, n)), 1.0));
    }
};
template <typename Ti, int M>
struct ColBlueDivPass {
    using CC = ColCfg<M, double, 2>;
    static constexpr int TPL = CC::TPL, LP = CC::LP, XC = CC::XC, OL = CC::OL, NT = CC::NT, LINES = CC::LINES;
    static constexpr int MINB = MinB<double, NT>::V;
    static constexpr size_t BUF = CC::SMEM;
    ColGeom c;
    const Cx<Ti>* p1;
    const Cx<Ti>* p2;
    const Cx<Ti>* p3;
    Cx<Ti>* q;
    Cx<Ti>* r;
    BlueTab<double> bt;
    int n1;
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int x = x0 + xi, o = o0 + oi;
        const bool on = x < c.nx && o < c.n3;
        Cx<double>* bA = reinterpret_cast<Cx<double>*>(smem) + (oi * XC + xi) * LP;
        Cx<double>* bB = bA + LINES * LP;
        blue_line<double, M, 0>(bA, t, bt, AccD<Ti>{col_acc<2>(const_cast<Cx<Ti>*>(p1), c, x, o, 0, on, 0)}, SmemLine<double>{bB});
        __syncthreads();
        const double k1 = (double)((x == n1 / 2) ? 0 : x);
        blue_line<double, M, 0>(bA, t, bt, AccD<Ti>{col_acc<2>(const_cast<Cx<Ti>*>(p2), c, x, o, 0, on, 0)},
                        DivCombineSt<Ti>{bB, AccD<Ti>{col_acc<2>(q, c, x, o, 0, on, 0)}, k1, bt.n});
        __syncthreads();
        blue_line<double, M, 0>(bA, t, bt, AccD<Ti>{col_acc<2>(const_cast<Cx<Ti>*>(p3), c, x, o, 0, on, 0)},
                        AccD<Ti>{col_acc<2>(r, c, x, o, 0, on, 0)});
    }
};

// ---------------------------------------------------------------------------------------------
// Spectral symbols applied in the x3 middle pass.  k = (k1, k2, k3) signed wavenumbers,
// kp = (k1', k2', k3') with the Nyquist zeroed.  `norm` = full inverse normalisation 2/M.
struct SymInfo {
    int reg;       // 1: a = |k|^2, 2: a = |k|^4
    double beta;
    double norm;
    int comp = 0;  // kind 6: the output component c
};

template <typename T>
__device__ __forceinline__ T sym_a(const SymInfo& s, T kk) { return s.reg == 1 ? kk : kk * kk; }

// kind 0: Y = norm * beta a(k) X                  (regulariser, Eq. 5e)
// kind 1: Y = norm * X / (beta a_hat(k))          (preconditioner; a_hat(0) = 1)
// kind 2: Y = norm * L_hat X                      (Leray, 3 -> 3)
// kind 3: Y = norm * L_hat X / (beta a_hat(k))    (isochoric preconditioner)
// kind 4: Y = norm * (beta a(k) V + L_hat B)      (isochoric matvec tail, 6 -> 3)
// kind 5: Y = norm * L_hat (beta a(k) V + B)      (isochoric gradient from the unprojected v, 6 -> 3)
// kind 6: Y = norm * (beta a(k) V_c + i k'_c D / |k'|^2)   (isochoric matvec tail per component c, 2 -> 1;
//         D = F[div b~]: L b~ = b~ - grad Lap^-1 div b~, whose b~ part is added in real space)
// kind 7: kind 6 for the three components in one pass (4 -> 3: V_0, V_1, V_2, D; MiddlePass::run7 reads
//         and transforms D once, then each V_c in turn through one input and one output line buffer)
// kind 8: kind 6 for the three components with D formed in the pass from the x2 stage of the data term
//         (ColDivPass): D = F3 Q + i k3' F3 R, Q and R in the I/O precision (MiddlePass::run_div; 3 -> 3 plus
//         the two spectra inq); kind 9: the same for one component (comp = SymInfo::comp; slabs)
template <typename T, int KIND>
struct Sym {
    static constexpr int NCI = (KIND <= 1 || KIND == 9) ? 1 : (KIND == 6 ? 2 : (KIND == 7 ? 4 : (KIND == 8 ? 3 : (KIND >= 4 ? 6 : 3))));
    static constexpr int NCO = (KIND <= 1 || KIND == 6 || KIND == 9) ? 1 : 3;
    static __device__ __forceinline__ void apply(const SymInfo& s, Cx<T>* x, int k1, int k2, int k3, int kp1, int kp2,
                                                 int kp3) {
        const T kk = T(k1) * T(k1) + T(k2) * T(k2) + T(k3) * T(k3);
        const T nrm = (T)s.norm;
        if (KIND == 6) {
            const T q1 = T(kp1), q2 = T(kp2), q3 = T(kp3);
            const T qq = q1 * q1 + q2 * q2 + q3 * q3;
            const T qc = s.comp == 0 ? q1 : (s.comp == 1 ? q2 : q3);
            const T f = (qq != T(0)) ? qc / qq : T(0);
            x[0] = scale(x[0], nrm * (T)s.beta * sym_a<T>(s, kk)) + mul_i(x[1], nrm * f);
            return;
        }
        if (KIND == 0) {
            x[0] = scale(x[0], nrm * (T)s.beta * sym_a<T>(s, kk));
        } else if (KIND == 1) {
            const T ah = (kk == T(0)) ? T(1) : sym_a<T>(s, kk);
            x[0] = scale(x[0], nrm / ((T)s.beta * ah));
        } else {
            const T q1 = T(kp1), q2 = T(kp2), q3 = T(kp3);
            const T qq = q1 * q1 + q2 * q2 + q3 * q3;
            Cx<T> b0, b1, b2;
            if (KIND == 5) {  // project beta a V + B
                const T ra = (T)s.beta * sym_a<T>(s, kk);
                b0 = scale(x[0], ra) + x[3];
                b1 = scale(x[1], ra) + x[4];
                b2 = scale(x[2], ra) + x[5];
            } else {
                Cx<T>* B = (KIND == 4) ? x + 3 : x;
                b0 = B[0];
                b1 = B[1];
                b2 = B[2];
            }
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

// Last forward stage of a one-component middle pass with a scalar symbol (KIND 0 / 1: a function of
// |k|^2 only): the symbol is applied to the stage's outputs in registers and the narrowed values go
// straight into the inverse's line, so no separate symbol sweep over shared memory is needed.  Same
// arithmetic as Sym<T, KIND>::apply (kk = (k1^2 + k2^2) + k3^2, factor evaluated in the same order).
template <typename Ti, typename To, int L, int KIND>
struct SymSt {
    Cx<To>* b;  // this line of the inverse's buffer
    Ti kk12;    // k1^2 + k2^2
    Ti nrm, beta;
    int reg;
    bool live;  // line inside the spectrum (dead lines are stored unscaled and never written out)
    __device__ __forceinline__ void st(int i, const Cx<Ti>& v) const {
        Cx<Ti> r = v;
        if (live) {
            const Ti k3 = (Ti)wavenum(i, L);
            const Ti kk = kk12 + k3 * k3;
            const Ti a = reg == 1 ? kk : kk * kk;
            if (KIND == 0) {
                r = scale(v, nrm * beta * a);
            } else {
                const Ti ah = (kk == Ti(0)) ? Ti(1) : a;
                r = scale(v, nrm / (beta * ah));
            }
        }
        b[P(i)] = cx<To>((To)r.re, (To)r.im);
    }
};

template <typename T, int NC>
struct SpecPtrs {
    Cx<T>* p[NC];
};

// x3 middle pass: forward FFT of NCI spectra along x3 in Ti, symbol in Ti, then the NCO results are
// narrowed to To in a second shared-memory region and transformed back in To (the inverse passes after
// the symbol may run in the I/O precision: their rounding is relative to the already-amplified signal).
template <typename Ti, typename To, int L, int KIND, bool PEER = false>
struct MiddlePass {
    using T = Ti;
    static constexpr int NCI = Sym<T, KIND>::NCI, NCO = Sym<T, KIND>::NCO;
    // line buffers in shared memory (kinds 8 / 9: one Ti buffer for V_c, two To buffers for Q / D and R / output)
    static constexpr int NCIS = KIND == 7 ? 2 : (KIND >= 8 ? 1 : NCI), NCOS = KIND == 7 ? 1 : (KIND >= 8 ? 2 : NCO);
    using CC = ColCfg<L, T, NCIS, (sizeof(T) == 8 && L >= 512) ? 128 : 0>;
    static constexpr int TPL = CC::TPL, LP = CC::LP, XC = CC::XC, OL = CC::OL, LINES = CC::LINES, NT = CC::NT;
    static constexpr int LPO = ColLP<L, To, XC>::V;  // stride of the To lines of the inverse
    static constexpr int TPLO = Tpl<L, To>::V;  // threads per inverse line (fp32: fewer than fp64)
    static constexpr int MINB = MinBMiddle<T, NT>::V;
    static constexpr size_t BUFI = CC::SMEM;
    static constexpr size_t BUFO = BUFI + (size_t)NCOS * LINES * LPO * sizeof(Cx<To>);
    static constexpr bool TWS = sizeof(T) == 4;
    static constexpr size_t BUF = BUFO + (TWS ? L * (sizeof(Cx<T>) + sizeof(Cx<To>)) : 0);  // + both twiddle tables
    ColGeom c;
    SpecPtrs<Ti, NCI> in;
    SpecPtrs<To, NCO> out;
    SpecPtrs<To, 2> inq;  // kinds 8 / 9: Q, R of ColDivPass
    SymInfo s;
    const Cx<Ti>* tw;
    const Cx<To>* two;  // inverse twiddles in To
    int64_t cs = 0;     // component stride of in / out (blockIdx.y = component; one-component symbols)
    PeerDst pd;         // PEER (one output): plane p goes to rank p >> pd.sh's receive buffer
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem);
        Cx<To>* so = reinterpret_cast<Cx<To>*>(smem + BUFI);
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int line = oi * XC + xi;
        const bool on = x0 + xi < c.nx && o0 + oi < c.n2;
        const Cx<T>* tw = tw_smem<T, L, NT, TWS>(this->tw, reinterpret_cast<Cx<T>*>(smem + BUFO));
        const Cx<To>* two = tw_smem<To, L, NT, TWS>(this->two, reinterpret_cast<Cx<To>*>(smem + BUFO + L * sizeof(Cx<T>)));
        if constexpr (KIND == 7) {
            run7(x0, o0, xi, t, oi, line, on, tw, two, sm, so);
        } else if constexpr (KIND >= 8) {
            run_div(x0, o0, xi, t, oi, line, on, tw, two, sm, so);
        } else {
            if constexpr (KIND <= 1) {  // scalar symbol fused into the last forward stage
                const int og = o0 + oi + c.k2off, n2g = c.n2g ? c.n2g : c.n2;
                const T k1 = (T)(x0 + xi), k2 = (T)wavenum(og, n2g);
                Cx<T>* buf = sm + line * LP;
                fft_line_io<T, L, -1, false, true>(
                    buf, t, tw, 1, col_acc<3>(in.p[0] + blockIdx.y * cs, c, x0 + xi, o0 + oi, 0, on, 0),
                    SymSt<T, To, L, KIND>{so + line * LPO, k1 * k1 + k2 * k2, (T)s.norm, (T)s.beta, s.reg, on});
            } else {
                forward_and_symbol(x0, o0, xi, t, oi, line, on, tw, sm, so);
            }
            inverse(x0, o0, two, so);
        }
    }
    __device__ __forceinline__ void forward_and_symbol(int x0, int o0, int xi, int t, int oi, int line, bool on,
                                                       const Cx<T>* tw, Cx<T>* sm, Cx<To>* so) const {
#pragma unroll
        for (int ci = 0; ci < NCI; ++ci) {
            Cx<T>* buf = sm + ci * LINES * LP + line * LP;
            fft_line_io<T, L, -1, false, true>(buf, t, tw, 1, col_acc<3>(in.p[ci], c, x0 + xi, o0 + oi, 0, on, 0),
                                               SmemLine<T>{buf});
        }
        // symbol: element (line, p): k1 = column index x (0..N1/2), k2 from the transverse index, k3 from p
        const int n1 = 2 * (c.nx - 1);
        for (int e = threadIdx.x; e < LINES * L; e += NT) {
            const int ln = e / L, p = e % L;
            const int lxi = ln % XC, loi = ln / XC;
            const int x = x0 + lxi, o = o0 + loi;
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
            for (int co = 0; co < NCO; ++co) so[co * LINES * LPO + ln * LPO + P(p)] = cx<To>((To)v[co].re, (To)v[co].im);
        }
        __syncthreads();
    }
    // kind 7: D's x3 spectrum once, then per component c: V_c forward, the kind-6 symbol of component c
    // (Sym<T, 6>::apply with comp = c: the same arithmetic, so the same bits), inverse to out.p[c]
    __device__ __forceinline__ void run7(int x0, int o0, int xi, int t, int oi, int line, bool on, const Cx<T>* tw,
                                         const Cx<To>* two, Cx<T>* sm, Cx<To>* so) const {
        Cx<T>* bV = sm;
        Cx<T>* bD = sm + LINES * LP;
        fft_line_io<T, L, -1, false, true>(bD + line * LP, t, tw, 1, col_acc<3>(in.p[3], c, x0 + xi, o0 + oi, 0, on, 0),
                                           SmemLine<T>{bD + line * LP});
        const int n1 = 2 * (c.nx - 1);
        for (int cc = 0; cc < 3; ++cc) {
            fft_line_io<T, L, -1, false, true>(bV + line * LP, t, tw, 1, col_acc<3>(in.p[cc], c, x0 + xi, o0 + oi, 0, on, 0),
                                               SmemLine<T>{bV + line * LP});
            SymInfo sc = s;
            sc.comp = cc;
            for (int e = threadIdx.x; e < LINES * L; e += NT) {
                const int ln = e / L, p = e % L;
                const int lxi = ln % XC, loi = ln / XC;
                const int x = x0 + lxi, o = o0 + loi;
                Cx<T> v[2] = {bV[ln * LP + P(p)], bD[ln * LP + P(p)]};
                if (x < c.nx && o < c.n2) {
                    const int og = o + c.k2off, n2g = c.n2g ? c.n2g : c.n2;
                    const int k1 = x, k2 = wavenum(og, n2g), k3 = wavenum(p, L);
                    const int kp1 = (x == n1 / 2) ? 0 : x, kp2 = wavenum_odd(og, n2g), kp3 = wavenum_odd(p, L);
                    Sym<T, 6>::apply(sc, v, k1, k2, k3, kp1, kp2, kp3);
                }
                so[ln * LPO + P(p)] = cx<To>((To)v[0].re, (To)v[0].im);
            }
            __syncthreads();
            inverse_one(cc, 0, x0, o0, two, so);
        }
    }
    // forward x3 transform in To of a To spectrum into line buffer set sb (the inverse's thread mapping)
    __device__ __forceinline__ void forward_o(const Cx<To>* src, Cx<To>* sb, int x0, int o0, const Cx<To>* two) const {
        constexpr int PER = NT / TPLO;  // lines per round
        static_assert(NT % TPLO == 0 && LINES % PER == 0, "forward_o thread mapping");
#pragma unroll
        for (int l0 = 0; l0 < LINES; l0 += PER) {
            const int lxi = threadIdx.x % XC;
            const int rr = threadIdx.x / XC;
            const int lt = rr % TPLO, loi = l0 / XC + rr / TPLO;
            const int ln = loi * XC + lxi;
            const bool lon = x0 + lxi < c.nx && o0 + loi < c.n2;
            Cx<To>* buf = sb + ln * LPO;
            fft_line_io<To, L, -1, false, true>(buf, lt, two, 1,
                                                col_acc<3>(const_cast<Cx<To>*>(src), c, x0 + lxi, o0 + loi, 0, lon, 0),
                                                SmemLine<To>{buf});
        }
    }
    // kinds 8 / 9: D = F3 Q + i k3' F3 R once (To), then per component c: V_c forward (Ti), the kind-6 symbol
    // of component c with D widened to Ti, narrowed into R's buffer, inverse to the output
    __device__ __forceinline__ void run_div(int x0, int o0, int xi, int t, int oi, int line, bool on, const Cx<T>* tw,
                                            const Cx<To>* two, Cx<T>* sm, Cx<To>* so) const {
        Cx<To>* bQ = so;
        Cx<To>* bR = so + LINES * LPO;
        forward_o(inq.p[0], bQ, x0, o0, two);
        forward_o(inq.p[1], bR, x0, o0, two);
        for (int e = threadIdx.x; e < LINES * L; e += NT) {
            const int ln = e / L, p = e % L;
            const To k3 = (To)wavenum_odd(p, L);
            bQ[ln * LPO + P(p)] = bQ[ln * LPO + P(p)] + mul_i(bR[ln * LPO + P(p)], k3);
        }
        __syncthreads();
        const int n1 = 2 * (c.nx - 1);
        constexpr int NCC = KIND == 8 ? 3 : 1;
        for (int ci = 0; ci < NCC; ++ci) {
            const Cx<T>* vin = KIND == 8 ? in.p[ci] : in.p[0] + blockIdx.y * cs;
            fft_line_io<T, L, -1, false, true>(sm + line * LP, t, tw, 1,
                                               col_acc<3>(const_cast<Cx<T>*>(vin), c, x0 + xi, o0 + oi, 0, on, 0),
                                               SmemLine<T>{sm + line * LP});
            SymInfo sc = s;
            sc.comp = KIND == 8 ? ci : s.comp;
            for (int e = threadIdx.x; e < LINES * L; e += NT) {
                const int ln = e / L, p = e % L;
                const int lxi = ln % XC, loi = ln / XC;
                const int x = x0 + lxi, o = o0 + loi;
                const Cx<To> d = bQ[ln * LPO + P(p)];
                Cx<T> v[2] = {sm[ln * LP + P(p)], cx<T>((T)d.re, (T)d.im)};
                if (x < c.nx && o < c.n2) {
                    const int og = o + c.k2off, n2g = c.n2g ? c.n2g : c.n2;
                    const int k1 = x, k2 = wavenum(og, n2g), k3 = wavenum(p, L);
                    const int kp1 = (x == n1 / 2) ? 0 : x, kp2 = wavenum_odd(og, n2g), kp3 = wavenum_odd(p, L);
                    Sym<T, 6>::apply(sc, v, k1, k2, k3, kp1, kp2, kp3);
                }
                bR[ln * LPO + P(p)] = cx<To>((To)v[0].re, (To)v[0].im);
            }
            __syncthreads();
            inverse_one(KIND == 8 ? ci : 0, 1, x0, o0, two, so);
        }
    }
    __device__ __forceinline__ void inverse(int x0, int o0, const Cx<To>* two, Cx<To>* so) const {
#pragma unroll
        for (int co = 0; co < NCO; ++co) inverse_one(co, co, x0, o0, two, so);
    }
    // inverse of line buffer set `cb` to output co
    __device__ __forceinline__ void inverse_one(int co, int cb, int x0, int o0, const Cx<To>* two, Cx<To>* so) const {
        // inverse lines: the CTA's NT threads cover LINES lines of TPLO threads in NT / (LINES * TPLO) rounds
        static_assert(NT % TPLO == 0, "inverse thread mapping");
        constexpr int PER = NT / TPLO;  // lines per round
        {
#pragma unroll
            for (int l0 = 0; l0 < LINES; l0 += PER) {
                // thread -> (column, t, line) with columns fastest, as in col_thread
                const int lxi = threadIdx.x % XC;
                const int rr = threadIdx.x / XC;
                const int lt = rr % TPLO, loi = l0 / XC + rr / TPLO;
                const int ln = loi * XC + lxi;
                const bool act = ln < LINES;
                const bool lon = act && x0 + lxi < c.nx && o0 + loi < c.n2;
                Cx<To>* buf = so + cb * LINES * LPO + (act ? ln : 0) * LPO;
                if constexpr (PEER) {  // rank q's chunk: [i3 - q n3][line][x] (the split layout of the inverse x2 pass)
                    const int mk = (1 << pd.sh) - 1;
                    PeerAcc<To> pa{pd.pws, pd.boff, (int64_t)(o0 + loi) * c.W + x0 + lxi, (int64_t)c.n2 * c.W, pd.sh, mk, lon};
                    fft_line_io<To, L, +1, true, false>(buf, lt, two, 1, SmemLine<To>{buf}, pa);
                } else {
                    fft_line_io<To, L, +1, true, false>(buf, lt, two, 1, SmemLine<To>{buf},
                                                        col_acc<3>(out.p[co] + blockIdx.y * cs, c, x0 + lxi, o0 + loi, 0, lon, 0));
                }
            }
        }
    }
};

// x3 middle pass of an x3 extent that is not a power of two (one rank): every line of every input goes
// through a Bluestein forward transform (fp64) into its own shared-memory line, the symbol is applied
// there (Sym<double, KIND>, the same expressions as MiddlePass), and every output line goes back through
// a Bluestein inverse; I/O in the spectra's types.  Kinds 0 / 1 (scalar, components by blockIdx.y),
// 2 / 3 / 5 (coupled) and 8 (the isochoric data term from ColDivPass's Q, R: D = F3 Q + i k3' F3 R).
template <int M, int NB>
struct BlueMidCfg {
    static constexpr int TPL = Tpl<M, double>::V;
    static constexpr int XC = NB <= 2 ? 4 : 2;
    static constexpr int LW = ColLP<M, double, XC>::V;       // work line (M points)
    static constexpr int LD = M / 2 + M / 32 + 2;              // data line: n3 <= M / 2 points, padded by P()
    static constexpr size_t PER = (size_t)(NB * LD + LW) * sizeof(Cx<double>);
    static constexpr int OLT = (128 / (XC * TPL)) > 0 ? 128 / (XC * TPL) : 1;
    static constexpr int OLS = (int)((96 * 1024) / (XC * PER)) > 0 ? (int)((96 * 1024) / (XC * PER)) : 1;
    static constexpr int OL = OLT < OLS ? OLT : OLS;
    static constexpr int LINES = XC * OL, NT = XC * OL * TPL;
    static constexpr size_t SMEM = LINES * PER;
};
template <typename Ti, typename To, int M, int KIND>
struct BlueMiddlePass {
    static constexpr int NCI = Sym<double, KIND>::NCI, NCO = Sym<double, KIND>::NCO;
    static constexpr int NB = KIND == 8 ? 5 : NCI;  // data lines per transverse line
    using CC = BlueMidCfg<M, NB>;
    static constexpr int TPL = CC::TPL, XC = CC::XC, OL = CC::OL, NT = CC::NT, LINES = CC::LINES;
    static constexpr int MINB = 1;
    static constexpr size_t BUF = CC::SMEM;
    ColGeom c;
    SpecPtrs<Ti, NCI> in;
    SpecPtrs<To, NCO> out;
    SpecPtrs<To, 2> inq;
    SymInfo s;
    BlueTab<double> bt;
    int64_t cs = 0;
    __device__ __forceinline__ Cx<double>* dline(unsigned char* smem, int b, int ln) const {
        return reinterpret_cast<Cx<double>*>(smem) + (size_t)LINES * CC::LW + ((size_t)b * LINES + ln) * CC::LD;
    }
    __device__ __forceinline__ void run(int tile, unsigned char* smem) const {
        int x0, o0, xi, t, oi;
        col_origin<XC, OL>(c, tile, x0, o0);
        col_thread<XC, TPL>(xi, t, oi);
        const int x = x0 + xi, o = o0 + oi, ln = oi * XC + xi;
        const bool on = x < c.nx && o < c.n2;
        const int n = bt.n;
        Cx<double>* work = reinterpret_cast<Cx<double>*>(smem) + (size_t)ln * CC::LW;
        const int64_t off = (KIND <= 1) ? blockIdx.y * cs : 0;
#pragma unroll 1
        for (int b = 0; b < NB; ++b) {
            if (b < NCI) {
                blue_line<double, M, 0>(work, t, bt, AccD<Ti>{col_acc<3>(in.p[b] + off, c, x, o, 0, on, 0)},
                                        SmemLine<double>{dline(smem, b, ln)});
            } else {
                blue_line<double, M, 0>(work, t, bt, AccD<To>{col_acc<3>(inq.p[b - NCI], c, x, o, 0, on, 0)},
                                        SmemLine<double>{dline(smem, b, ln)});
            }
            __syncthreads();
        }
        const int n1 = 2 * (c.nx - 1);
        for (int e = threadIdx.x; e < LINES * n; e += NT) {
            const int l = e / n, p = e % n;
            const int lx = x0 + l % XC, lo = o0 + l / XC;
            Cx<double> v[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) v[b] = dline(smem, b, l)[P(p)];
            if (lx < c.nx && lo < c.n2) {
                const int og = lo + c.k2off, n2g = c.n2g ? c.n2g : c.n2;
                const int k1 = lx, k2 = wavenum(og, n2g), k3 = wavenum(p, n);
                const int kp1 = (lx == n1 / 2) ? 0 : lx, kp2 = wavenum_odd(og, n2g), kp3 = wavenum_odd(p, n);
                if constexpr (KIND == 8) {
                    const Cx<double> d = v[3] + mul_i(v[4], (double)kp3);
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) {
                        SymInfo sc = s;
                        sc.comp = cc;
                        Cx<double> w2[2] = {v[cc], d};
                        Sym<double, 6>::apply(sc, w2, k1, k2, k3, kp1, kp2, kp3);
                        v[cc] = w2[0];
                    }
                } else {
                    Sym<double, KIND>::apply(s, v, k1, k2, k3, kp1, kp2, kp3);
                }
            }
#pragma unroll
            for (int b = 0; b < NCO; ++b) dline(smem, b, l)[P(p)] = v[b];
        }
        __syncthreads();
#pragma unroll 1
        for (int b = 0; b < NCO; ++b) {
            blue_line<double, M, 1>(work, t, bt, SmemLine<double>{dline(smem, b, ln)},
                                    AccD<To>{col_acc<3>(out.p[b] + off, c, x, o, 0, on, 0)});
            __syncthreads();
        }
    }
};

// Line FFT with an arbitrary shared-memory line accessor, in place (source = intermediate = line).
template <typename T, int L, int DIR, int TPL, int R, int Ns, bool DST_SMEM, class LineT, class Dst>
__device__ __forceinline__ void stages_rest_l(const LineT& line, int t, const Cx<T>* __restrict__ tw, int tws,
                                              const Dst& dst) {
    if constexpr (Ns * R >= L) {
        stage_io<T, L, L / Ns, Ns, DIR, TPL, DST_SMEM>(t, tw, tws, line, dst);
        if (DST_SMEM) __syncthreads();
    } else {
        stage_io<T, L, R, Ns, DIR, TPL, true>(t, tw, tws, line, line);
        __syncthreads();
        stages_rest_l<T, L, DIR, TPL, R, Ns * R, DST_SMEM>(line, t, tw, tws, dst);
    }
}
template <typename T, int L, int DIR, bool DST_SMEM, class LineT, class Dst>
__device__ __forceinline__ void fft_line_inplace(const LineT& line, int t, const Cx<T>* __restrict__ tw, int tws,
                                                 const Dst& dst) {
    constexpr int TPL = Tpl<L, T>::V, R = Tpl<L, T>::R;
    if constexpr (L <= R) {
        stage_io<T, L, L, 1, DIR, TPL, true>(t, tw, tws, line, dst);
        if (DST_SMEM) __syncthreads();
    } else {
        stage_io<T, L, R, 1, DIR, TPL, true>(t, tw, tws, line, line);
        __syncthreads();
        stages_rest_l<T, L, DIR, TPL, R, R, DST_SMEM>(line, t, tw, tws, dst);
    }
}
// line xi of a staged column tile: element p at row p (row = XC consecutive columns, 128 bytes)
template <typename T, int XC>
struct StgLine {
    Cx<T>* b;
    __device__ __forceinline__ Cx<T> ld(int i) const { return b[i * XC]; }
    __device__ __forceinline__ void st(int i, const Cx<T>& v) const { b[i * XC] = v; }
};

// x3 middle pass with a scalar symbol (KIND 0 / 1), tiles fetched by the tensor-map TMA engine: one
// cp.async.bulk.tensor request per tile (XC columns x one k2 line x all L planes, 32 KB) lands as
// [p][XC columns] rows of 128 bytes; the forward FFT in Ti, the symbol (in the last forward stage) and
// the fp32 inverse all run in place there (a narrowed fp32 value takes the first half of its fp64
// slot).  Persistent CTAs, two stages: tile i+1 is in flight while tile i is transformed.  The 4-D
// tensor map is (2 W scalars, n2, n3, components).
template <typename Ti, int L, int KIND>
struct MiddleTma {
    using T = Ti;
    using CC = ColCfg<L, T, 1, ColCap<L, T>::V>;
    static constexpr int TPL = CC::TPL, XC = CC::XC, NT = CC::NT;
    static_assert(CC::OL == 1 && XC * sizeof(Cx<T>) == 128, "one 128-byte row per plane");
    static_assert(Tpl<L, float>::V == TPL, "the fp32 inverse keeps the thread -> (column, t) map");
    static constexpr int MINB = MinBMiddle<T, NT>::V;
    static constexpr size_t STG = (size_t)L * XC * sizeof(Cx<T>);
    static constexpr bool TWS = sizeof(T) == 4;  // fp32: twiddles in shared memory (fp64: L1, as MiddlePass)
    static constexpr size_t BUF = 128 + 2 * STG + (TWS ? L * sizeof(Cx<T>) : 0);
    static constexpr int XO = (int)(sizeof(Cx<T>) / sizeof(Cx<float>));  // fp32 slots per Ti slot
    ColGeom c;
    Cx<float>* out;
    int64_t cs;  // output component stride
    SymInfo s;
    const Cx<T>* tw;
    const Cx<float>* two;
    __device__ __forceinline__ void origin(int tile, int& x0, int& o) const {
        const int nxb = (c.nx + XC - 1) / XC;
        x0 = (tile % nxb) * XC;
        o = tile / nxb;
    }
};

// the last forward stage of a staged line: symbol in registers, narrowed in place (first half of the slot)
template <typename T, int L, int RS, int KIND>
struct SymStStg {
    Cx<float>* b;  // line base as fp32 slots, row stride RS fp32 slots
    T kk12, nrm, beta;
    int reg;
    bool live;
    __device__ __forceinline__ void st(int i, const Cx<T>& v) const {
        Cx<T> r = v;
        if (live) {
            const T k3 = (T)wavenum(i, L);
            const T kk = kk12 + k3 * k3;
            const T a = reg == 1 ? kk : kk * kk;
            if (KIND == 0) {
                r = scale(v, nrm * beta * a);
            } else {
                const T ah = (kk == T(0)) ? T(1) : a;
                r = scale(v, nrm / (beta * ah));
            }
        }
        b[i * RS] = cx<float>((float)r.re, (float)r.im);
    }
};

template <typename T> struct TmaType;
template <> struct TmaType<float> { static constexpr CUtensorMapDataType V = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; };
template <> struct TmaType<double> { static constexpr CUtensorMapDataType V = CU_TENSOR_MAP_DATA_TYPE_FLOAT64; };

__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

template <typename Ti, int L, int KIND>
__global__ void __launch_bounds__(MiddleTma<Ti, L, KIND>::NT, MiddleTma<Ti, L, KIND>::MINB)
    k_middle_tma(const __grid_constant__ CUtensorMap tmap, MiddleTma<Ti, L, KIND> pass, int ntiles) {
    using P = MiddleTma<Ti, L, KIND>;
    using T = Ti;
    constexpr int XC = P::XC, TPL = P::TPL, XO = P::XO;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* stg = smem_raw + 128;
    const Cx<T>* tw = pass.tw;
    const Cx<float>* two = pass.two;
    if constexpr (P::TWS) {
        Cx<T>* tws = reinterpret_cast<Cx<T>*>(stg + 2 * P::STG);
        for (int i = threadIdx.x; i < L; i += P::NT) tws[i] = pass.tw[i];
        tw = tws;
        two = reinterpret_cast<const Cx<float>*>(tws);  // fp32: the same table
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int tile, int st) {
        int x0, o;
        pass.origin(tile, x0, o);
        mbar_expect(&bar[st], (unsigned)P::STG);
        tma_load_4d(stg + st * P::STG, &tmap, 2 * x0, o, 0, blockIdx.y, &bar[st]);
    };
    int tile = blockIdx.x;
    if (threadIdx.x == 0 && tile < ntiles) issue(tile, 0);
    int xi, t, oi;
    col_thread<XC, TPL>(xi, t, oi);
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const int st = it & 1;
        if (threadIdx.x == 0 && tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, st ^ 1);
        mbar_wait(&bar[st], (unsigned)(it >> 1) & 1u);
        int x0, o;
        pass.origin(tile, x0, o);
        const int x = x0 + xi;
        const bool on = x < pass.c.nx && o < pass.c.n2;
        Cx<T>* base = reinterpret_cast<Cx<T>*>(stg + st * P::STG);
        const StgLine<T, XC> line{base + xi};
        Cx<float>* fb = reinterpret_cast<Cx<float>*>(base) + XO * xi;  // fp32 view of the line
        const int og = o + pass.c.k2off, n2g = pass.c.n2g ? pass.c.n2g : pass.c.n2;
        const T k1 = (T)x, k2 = (T)wavenum(og, n2g);
        fft_line_inplace<T, L, -1, true>(line, t, tw, 1,
                                         SymStStg<T, L, XO * XC, KIND>{fb, k1 * k1 + k2 * k2, (T)pass.s.norm,
                                                                       (T)pass.s.beta, pass.s.reg, on});
        fft_line_inplace<float, L, +1, false>(StgLine<float, XO * XC>{fb}, t, two, 1,
                                              col_acc<3, float, false>(pass.out + blockIdx.y * pass.cs, pass.c, x, o, 0, on, 0));
        // generic-proxy writes to the stage (the in-place transforms) must be ordered before the
        // async-proxy (TMA) refill of the same buffer: every writer fences, then the barrier
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();  // the stage is refilled two iterations later
    }
}

// One CTA per tile of a pass.
template <class PassT>
__global__ void __launch_bounds__(PassT::NT, PassT::MINB) k_stream(PassT pass) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    pass.run(blockIdx.x, smem_raw);
}

}  // namespace dr
