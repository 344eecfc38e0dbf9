// fft.cuh -- shared-memory Stockham FFT passes for the spectral operators (§III-B1,
// L303 §III-C1).  Every pass streams a field once from HBM into shared memory, transforms whole
// lines there (radix-16 register butterflies, padded smem to avoid bank conflicts, fp32/fp64
// twiddles from a table built in double precision on the host) and streams it back.
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
    static constexpr int TPL = (L >= 16) ? L / 16 : 1;  // threads per line
    static constexpr int LP = L + L / 16 + 2;           // padded line length (holds index L for r2c)
};
// Row passes: RB rows per CTA, ~256 threads for fp32 compute and ~128 for fp64 (register footprint of
// the radix-16 butterflies doubles) so several CTAs fit per SM.
template <int L, typename Tc>
struct RowCfg {
    static constexpr int NTT = sizeof(Tc) == 8 ? 128 : 256;
    static constexpr int RB = (NTT / LineGeom<L>::TPL) > 0 ? NTT / LineGeom<L>::TPL : 1;
    static constexpr int NT = RB * LineGeom<L>::TPL;
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

// One Stockham autosort stage of radix R (Ns = product of the previous radices) on a line of
// length L held in padded shared memory.  Each of the TPL threads of the line owns 16 values
// (L/R/TPL butterflies).  tw: table of e^{-2 pi i m / (L*tws)}, m < L*tws.
template <typename T, int L, int R, int Ns, int DIR>
__device__ __forceinline__ void stockham_stage(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws) {
    constexpr int TPL = LineGeom<L>::TPL;
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

// Whole-line FFT (in place, padded layout).  Radix plan: 16 x 16 x ... x r.
// Every thread of the CTA must call this (it contains __syncthreads).
template <typename T, int L, int DIR>
__device__ __forceinline__ void fft_line(Cx<T>* buf, int t, const Cx<T>* __restrict__ tw, int tws) {
    if constexpr (L <= 16) {
        stockham_stage<T, L, L, 1, DIR>(buf, t, tw, tws);
    } else if constexpr (L <= 256) {
        stockham_stage<T, L, 16, 1, DIR>(buf, t, tw, tws);
        stockham_stage<T, L, L / 16, 16, DIR>(buf, t, tw, tws);
    } else {
        stockham_stage<T, L, 16, 1, DIR>(buf, t, tw, tws);
        stockham_stage<T, L, 16, 16, DIR>(buf, t, tw, tws);
        stockham_stage<T, L, L / 256, 256, DIR>(buf, t, tw, tws);
    }
}

// ---------------------------------------------------------------------------------------------
// real <-> half-complex post/pre-processing of a row of N = 2L reals packed as L complex
// z_n = x_{2n} + i x_{2n+1}.  After the forward L-point FFT Z, X_k (k = 0..L) of the N-point DFT:
//   E = (Z_k + conj Z_{L-k})/2, O = (Z_k - conj Z_{L-k})/(2i), X_k = E + W^k O, X_{L-k} = conj(E - W^k O),
// W = e^{-2 pi i/N}.  Pairs (k, L-k) are handled by one thread, so the update is in place.
template <typename T, int L>
__device__ __forceinline__ void r2c_post(Cx<T>* buf, int t, const Cx<T>* __restrict__ twN) {
    constexpr int TPL = LineGeom<L>::TPL;
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
template <typename T, int L>
__device__ __forceinline__ void c2r_pre(Cx<T>* buf, int t, const Cx<T>* __restrict__ twN) {
    constexpr int TPL = LineGeom<L>::TPL;
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

// ---------------------------------------------------------------------------------------------
// Row pass: x1-derivative of real rows ("N2 N3 1D FFTs across the first coordinate,
// diagonal scaling, and then the same number of inverse FFTs").  out = acc*out + d f/dx1.
template <typename T, int L>
__global__ void __launch_bounds__(RowCfg<L, T>::NT) k_row_deriv(Grid g, const T* __restrict__ f, T* __restrict__ out,
                                                   int accumulate, const Cx<T>* __restrict__ twN) {
    constexpr int TPL = LineGeom<L>::TPL, LP = LineGeom<L>::LP;
    constexpr int RB = RowCfg<L, T>::RB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem_raw);
    const int64_t nrows = (int64_t)g.n2 * g.n3;
    const int64_t row0 = (int64_t)blockIdx.x * RB;
    const Cx<T>* src = reinterpret_cast<const Cx<T>*>(f) + row0 * L;
    const int nvalid = (int)((nrows - row0) < RB ? (nrows - row0) : RB);
    for (int e = threadIdx.x; e < nvalid * L; e += blockDim.x) sm[(e / L) * LP + P(e % L)] = src[e];
    __syncthreads();
    const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
    Cx<T>* buf = sm + line * LP;
    fft_line<T, L, -1>(buf, t, twN, 2);
    r2c_post<T, L>(buf, t, twN);
    // X_k *= i k'_1 / L  (k = 0..L; Nyquist k = L is zeroed, reading A2; 1/L normalises the c2r)
    for (int k = t; k <= L; k += TPL) {
        const T kk = (k == L) ? T(0) : T(k);
        buf[P(k)] = mul_i(buf[P(k)], kk / T(L));
    }
    __syncthreads();
    c2r_pre<T, L>(buf, t, twN);
    fft_line<T, L, +1>(buf, t, twN, 2);
    Cx<T>* dst = reinterpret_cast<Cx<T>*>(out) + row0 * L;
    for (int e = threadIdx.x; e < nvalid * L; e += blockDim.x) {
        Cx<T> v = sm[(e / L) * LP + P(e % L)];
        if (accumulate) { const Cx<T> o = dst[e]; v = v + o; }
        dst[e] = v;
    }
}

// Row pass: real rows (type Ti) -> half-spectrum rows (r2c along x1) computed and stored in Tc,
// spectrum row stride g.n1p.  Ti = float, Tc = double keeps the forward spectrum exact enough for the
// high-wavenumber amplification of beta*A.
template <typename Ti, typename Tc, int L>
__global__ void __launch_bounds__(RowCfg<L, Tc>::NT) k_row_r2c(Grid g, const Ti* __restrict__ f, Cx<Tc>* __restrict__ spec,
                                                 const Cx<Tc>* __restrict__ twN) {
    constexpr int TPL = LineGeom<L>::TPL, LP = LineGeom<L>::LP;
    constexpr int RB = RowCfg<L, Tc>::RB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx<Tc>* sm = reinterpret_cast<Cx<Tc>*>(smem_raw);
    const int64_t nrows = (int64_t)g.n2 * g.n3;
    const int64_t row0 = (int64_t)blockIdx.x * RB;
    const Cx<Ti>* src = reinterpret_cast<const Cx<Ti>*>(f) + row0 * L;
    const int nvalid = (int)((nrows - row0) < RB ? (nrows - row0) : RB);
    for (int e = threadIdx.x; e < nvalid * L; e += blockDim.x) {
        const Cx<Ti> v = src[e];
        sm[(e / L) * LP + P(e % L)] = cx<Tc>((Tc)v.re, (Tc)v.im);
    }
    __syncthreads();
    const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
    Cx<Tc>* buf = sm + line * LP;
    fft_line<Tc, L, -1>(buf, t, twN, 2);
    r2c_post<Tc, L>(buf, t, twN);
    constexpr int NC = L + 1;
    for (int e = threadIdx.x; e < nvalid * NC; e += blockDim.x) {
        const int r = e / NC, k = e % NC;
        spec[(row0 + r) * g.n1p + k] = sm[r * LP + P(k)];
    }
}

// Row pass epilogue for the c2r inverse: out = x (+ add)
template <typename T>
struct RowOut {
    T* out;
    const T* add;  // nullable: field added after the inverse (b~ in the non-isochoric matvec)
};

// Row pass: half-spectrum rows -> real rows (c2r along x1) in T with epilogue out = x + add.
// The spectrum already carries the full inverse normalisation.
template <typename T, int L>
__global__ void __launch_bounds__(RowCfg<L, T>::NT) k_row_c2r(Grid g, const Cx<T>* __restrict__ spec, RowOut<T> epi,
                                                 const Cx<T>* __restrict__ twN) {
    constexpr int TPL = LineGeom<L>::TPL, LP = LineGeom<L>::LP;
    constexpr int RB = RowCfg<L, T>::RB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem_raw);
    const int64_t nrows = (int64_t)g.n2 * g.n3;
    const int64_t row0 = (int64_t)blockIdx.x * RB;
    const int nvalid = (int)((nrows - row0) < RB ? (nrows - row0) : RB);
    constexpr int NC = L + 1;
    for (int e = threadIdx.x; e < nvalid * NC; e += blockDim.x) {
        const int r = e / NC, k = e % NC;
        sm[r * LP + P(k)] = spec[(row0 + r) * g.n1p + k];
    }
    __syncthreads();
    const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
    Cx<T>* buf = sm + line * LP;
    c2r_pre<T, L>(buf, t, twN);
    fft_line<T, L, +1>(buf, t, twN, 2);
    Cx<T>* dst = reinterpret_cast<Cx<T>*>(epi.out) + row0 * L;
    const Cx<T>* add = epi.add ? reinterpret_cast<const Cx<T>*>(epi.add) + row0 * L : nullptr;
    for (int e = threadIdx.x; e < nvalid * L; e += blockDim.x) {
        Cx<T> v = sm[(e / L) * LP + P(e % L)];
        if (add) v = v + add[e];
        dst[e] = v;
    }
}

// ---------------------------------------------------------------------------------------------
// Column passes along x2 (AX = 2) or x3 (AX = 3) of a complex array with W complex columns per row
// (W = n1p for spectra, N1/2 for a real field read as pairs) and extents (W, n2, n3).
// A CTA owns XC consecutive columns x OL lines of the other transverse axis.
struct ColGeom {
    int W;      // row stride in complex elements
    int nx;     // valid columns (x < nx)
    int n2, n3;
};

template <int AX>
__device__ __forceinline__ int64_t col_addr(const ColGeom& c, int x, int other, int p) {
    if (AX == 2) return ((int64_t)other * c.n2 + p) * c.W + x;  // other = i3, p = i2
    return ((int64_t)p * c.n2 + other) * c.W + x;               // other = i2, p = i3
}

// CTA shape of a column pass: XC columns x OL transverse lines, TPL threads per line.  OL is chosen for
// ~256 threads but capped so that NC components of ES-byte complex values fit in ~72 KB of smem.
template <int L, int XC, int NC = 1, int ES = 16>
struct ColCfg {
    static constexpr int TPL = LineGeom<L>::TPL;
    static constexpr int NTT = ES == 16 ? 128 : 256;  // fp64 compute: fewer threads, more CTAs per SM
    static constexpr int OLT = (XC * TPL >= NTT) ? 1 : NTT / (XC * TPL);
    static constexpr int MAXL = (72 * 1024) / (NC * LineGeom<L>::LP * ES);
    static constexpr int OLS = (MAXL / XC) >= 1 ? MAXL / XC : 1;
    static constexpr int OL = OLT < OLS ? OLT : OLS;
    static constexpr int NT = XC * OL * TPL;
    static constexpr int LINES = XC * OL;
};

template <typename T, int L, int XC, int OL, int AX>
__device__ __forceinline__ void col_load(Cx<T>* sm, const Cx<T>* __restrict__ src, const ColGeom& c, int x0, int o0,
                                         int nother) {
    constexpr int LP = LineGeom<L>::LP;
    for (int e = threadIdx.x; e < XC * L * OL; e += blockDim.x) {
        const int xi = e % XC, p = (e / XC) % L, oi = e / (XC * L);
        const int x = x0 + xi, o = o0 + oi;
        Cx<T> v = cx(T(0), T(0));
        if (x < c.nx && o < nother) v = src[col_addr<AX>(c, x, o, p)];
        sm[(oi * XC + xi) * LP + P(p)] = v;
    }
}

template <typename T, int L, int XC, int OL, int AX, bool ACC, typename To = T>
__device__ __forceinline__ void col_store(const Cx<T>* sm, Cx<To>* __restrict__ dst, const ColGeom& c, int x0, int o0,
                                          int nother) {
    constexpr int LP = LineGeom<L>::LP;
    for (int e = threadIdx.x; e < XC * L * OL; e += blockDim.x) {
        const int xi = e % XC, p = (e / XC) % L, oi = e / (XC * L);
        const int x = x0 + xi, o = o0 + oi;
        if (x < c.nx && o < nother) {
            const Cx<T> w = sm[(oi * XC + xi) * LP + P(p)];
            Cx<To> v = cx<To>((To)w.re, (To)w.im);
            const int64_t a = col_addr<AX>(c, x, o, p);
            if (ACC) v = v + dst[a];
            dst[a] = v;
        }
    }
}

// Derivative along x2 / x3 of a real field (viewed as complex pairs): out (+)= d f / dx_AX.
template <typename T, int L, int XC, int AX>
__global__ void __launch_bounds__(ColCfg<L, XC, 1, sizeof(Cx<T>)>::NT) k_col_deriv(ColGeom c, const Cx<T>* __restrict__ src,
                                                                 Cx<T>* __restrict__ dst, int accumulate,
                                                                 const Cx<T>* __restrict__ tw) {
    constexpr int TPL = LineGeom<L>::TPL, LP = LineGeom<L>::LP;
    constexpr int OL = ColCfg<L, XC, 1, sizeof(Cx<T>)>::OL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem_raw);
    const int nxb = (c.nx + XC - 1) / XC;
    const int x0 = (blockIdx.x % nxb) * XC;
    const int o0 = (blockIdx.x / nxb) * OL;
    const int nother = (AX == 2) ? c.n3 : c.n2;
    col_load<T, L, XC, OL, AX>(sm, src, c, x0, o0, nother);
    __syncthreads();
    const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
    Cx<T>* buf = sm + line * LP;
    fft_line<T, L, -1>(buf, t, tw, 1);
    for (int k = t; k < L; k += TPL) {
        const T kp = (T)wavenum_odd(k, L);
        buf[P(k)] = mul_i(buf[P(k)], kp / T(L));
    }
    __syncthreads();
    fft_line<T, L, +1>(buf, t, tw, 1);
    if (accumulate) col_store<T, L, XC, OL, AX, true>(sm, dst, c, x0, o0, nother);
    else col_store<T, L, XC, OL, AX, false>(sm, dst, c, x0, o0, nother);
}

// Plain complex FFT of spectrum columns along x2 (forward DIR=-1 or inverse DIR=+1), in place.
template <typename T, int L, int XC, int DIR>
__global__ void __launch_bounds__(ColCfg<L, XC, 1, sizeof(Cx<T>)>::NT) k_col_fft(ColGeom c, Cx<T>* __restrict__ spec,
                                                               const Cx<T>* __restrict__ tw) {
    constexpr int TPL = LineGeom<L>::TPL, LP = LineGeom<L>::LP;
    constexpr int OL = ColCfg<L, XC, 1, sizeof(Cx<T>)>::OL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem_raw);
    const int nxb = (c.nx + XC - 1) / XC;
    const int x0 = (blockIdx.x % nxb) * XC;
    const int o0 = (blockIdx.x / nxb) * OL;
    col_load<T, L, XC, OL, 2>(sm, spec, c, x0, o0, c.n3);
    __syncthreads();
    const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
    fft_line<T, L, DIR>(sm + line * LP, t, tw, 1);
    col_store<T, L, XC, OL, 2, false>(sm, spec, c, x0, o0, c.n3);
}

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

// x3 middle pass: forward FFT of NCI spectra along x3, symbol, inverse FFT of NCO spectra, all in Ti;
// results are stored in To (the inverse passes after the symbol may run in the I/O precision: their
// rounding is relative to the already-amplified signal).
template <typename Ti, typename To, int L, int XC, int KIND>
__global__ void __launch_bounds__(ColCfg<L, XC, Sym<Ti, KIND>::NCI, sizeof(Cx<Ti>)>::NT) k_col_middle(ColGeom c, SpecPtrs<Ti, Sym<Ti, KIND>::NCI> in,
                                                                  SpecPtrs<To, Sym<Ti, KIND>::NCO> out, SymInfo s,
                                                                  const Cx<Ti>* __restrict__ tw) {
    using T = Ti;
    constexpr int TPL = LineGeom<L>::TPL, LP = LineGeom<L>::LP;
    constexpr int NCI = Sym<T, KIND>::NCI, NCO = Sym<T, KIND>::NCO;
    using CC = ColCfg<L, XC, NCI, sizeof(Cx<T>)>;
    constexpr int OL = CC::OL, LINES = CC::LINES;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx<T>* sm = reinterpret_cast<Cx<T>*>(smem_raw);
    const int nxb = (c.nx + XC - 1) / XC;
    const int x0 = (blockIdx.x % nxb) * XC;
    const int o0 = (blockIdx.x / nxb) * OL;
#pragma unroll
    for (int ci = 0; ci < NCI; ++ci) col_load<T, L, XC, OL, 3>(sm + ci * LINES * LP, in.p[ci], c, x0, o0, c.n2);
    __syncthreads();
    const int line = threadIdx.x / TPL, t = threadIdx.x % TPL;
#pragma unroll
    for (int ci = 0; ci < NCI; ++ci) fft_line<T, L, -1>(sm + ci * LINES * LP + line * LP, t, tw, 1);
    // symbol: element (line, p): k1 = column index x (0..N1/2), k2 from the transverse index, k3 from p
    const int n1 = 2 * (c.nx - 1);
    for (int e = threadIdx.x; e < LINES * L; e += blockDim.x) {
        const int ln = e / L, p = e % L;
        const int xi = ln % XC, oi = ln / XC;
        const int x = x0 + xi, o = o0 + oi;
        if (x >= c.nx || o >= c.n2) continue;
        Cx<T> v[NCI];
#pragma unroll
        for (int ci = 0; ci < NCI; ++ci) v[ci] = sm[ci * LINES * LP + ln * LP + P(p)];
        const int k1 = x, k2 = wavenum(o, c.n2), k3 = wavenum(p, L);
        const int kp1 = (x == n1 / 2) ? 0 : x, kp2 = wavenum_odd(o, c.n2), kp3 = wavenum_odd(p, L);
        Sym<T, KIND>::apply(s, v, k1, k2, k3, kp1, kp2, kp3);
#pragma unroll
        for (int co = 0; co < NCO; ++co) sm[co * LINES * LP + ln * LP + P(p)] = v[co];
    }
    __syncthreads();
#pragma unroll
    for (int co = 0; co < NCO; ++co) fft_line<T, L, +1>(sm + co * LINES * LP + line * LP, t, tw, 1);
#pragma unroll
    for (int co = 0; co < NCO; ++co)
        col_store<T, L, XC, OL, 3, false, To>(sm + co * LINES * LP, out.p[co], c, x0, o0, c.n2);
}

}  // namespace dr
