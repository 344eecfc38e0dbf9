/*
 * oracle/oracle.c -- fp64 CPU ORACLE for the Gauss-Newton Hessian matvec of arXiv 1608.03630.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA product path (paper_1608_03630_b200/csrc).
 *
 * Plain, slow, obviously correct: every primitive below is the textbook definition
 * written out in double precision, with citations into /root/reference/PAPER.md
 * ("P:Lnnn", plus the section / equation) and the discrete definitions D0-D14 of
 * SURVEY.md §8(c) (the readings of the paper this build commits to, listed in DESIGN.md).
 *
 * Grid (D0, §III-B1): N_a even >= 4, x_a = 2*pi*i_a/N_a, linear index
 * i1 + N1*(i2 + N2*i3) (x1 fastest).  Scalars: n1*n2*n3 doubles; vectors: 3 such blocks.
 *
 * OpenMP is used only to split independent outer loops (lines of an FFT, points of an
 * interpolation); it never changes the arithmetic of one output value.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

static const double PI = 3.14159265358979323846264338327950288;

/* --------------------------------------------------------------------------------------------
 * 1-D DFT  (D2, §III-B1: "Mappings between {rho_i} and {rho_hat_k} are done using the
 * forward and inverse Fast Fourier Transform").
 *   sign = -1 : a_k <- sum_j a_j exp(-2 pi i j k / n)      (forward)
 *   sign = +1 : a_k <- sum_j a_j exp(+2 pi i j k / n)      (inverse, unnormalised)
 * Power-of-two n: iterative radix-2 Cooley-Tukey; every twiddle is evaluated directly with
 * cos/sin of its own angle.  Other n: the O(n^2) definition.
 * ------------------------------------------------------------------------------------------ */
static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

static void dft_naive(cplx* a, int n, int sign, cplx* tmp) {
    for (int k = 0; k < n; ++k) {
        cplx s = 0;
        for (int j = 0; j < n; ++j) {
            double ang = sign * 2.0 * PI * (double)(((int64_t)j * k) % n) / (double)n;
            s += a[j] * (cos(ang) + I * sin(ang));
        }
        tmp[k] = s;
    }
    memcpy(a, tmp, sizeof(cplx) * (size_t)n);
}

static void fft1d(cplx* a, int n, int sign, cplx* tmp) {
    if (!is_pow2(n)) { dft_naive(a, n, sign, tmp); return; }
    /* bit-reversal permutation */
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { cplx t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (int len = 2; len <= n; len <<= 1) {
        int half = len >> 1;
        for (int i = 0; i < n; i += len) {
            for (int j = 0; j < half; ++j) {
                double ang = sign * 2.0 * PI * (double)j / (double)len;
                cplx w = cos(ang) + I * sin(ang);
                cplx u = a[i + j];
                cplx t = a[i + j + half] * w;
                a[i + j] = u + t;
                a[i + j + half] = u - t;
            }
        }
    }
}

/* 3-D DFT of a complex field in place, one axis at a time (separability of the DFT). */
void or_fft3(int n1, int n2, int n3, cplx* a, int sign) {
    const int n[3] = {n1, n2, n3};
    const int64_t stride[3] = {1, n1, (int64_t)n1 * n2};
    for (int ax = 0; ax < 3; ++ax) {
        const int L = n[ax];
        const int64_t nlines = (int64_t)n1 * n2 * n3 / L;
        #pragma omp parallel
        {
            cplx* line = (cplx*)malloc(sizeof(cplx) * (size_t)L);
            cplx* tmp = (cplx*)malloc(sizeof(cplx) * (size_t)L);
            #pragma omp for schedule(static)
            for (int64_t l = 0; l < nlines; ++l) {
                /* decompose the line index into the two coordinates orthogonal to ax */
                int64_t base;
                if (ax == 0) base = l * n1;
                else if (ax == 1) base = (l / n1) * (int64_t)n1 * n2 + (l % n1);
                else base = l;
                for (int p = 0; p < L; ++p) line[p] = a[base + p * stride[ax]];
                fft1d(line, L, sign, tmp);
                for (int p = 0; p < L; ++p) a[base + p * stride[ax]] = line[p];
            }
            free(line);
            free(tmp);
        }
    }
}

/* --------------------------------------------------------------------------------------------
 * Wavenumbers (D2/D3): index i on an axis of length N carries k = i for i <= N/2, else i - N,
 * i.e. k in {-N/2+1, ..., N/2}.  First-order symbols use k' = k if |k| < N/2 else 0
 * (Nyquist zeroed: SURVEY §8(c) A2); even-order symbols use the full k.
 * ------------------------------------------------------------------------------------------ */
static double wavenum(int i, int N) { return (i <= N / 2) ? (double)i : (double)(i - N); }
static double wavenum_odd(int i, int N) {
    double k = wavenum(i, N);
    return (fabs(k) < 0.5 * N) ? k : 0.0;
}

/* Multiply a complex spectrum by a scalar symbol sym(k1,k2,k3) given by `kind`. */
enum { SYM_DX1 = 0, SYM_DX2 = 1, SYM_DX3 = 2, SYM_LAP = 3, SYM_BIHARM = 4 };

static cplx symbol(int kind, double k1, double k2, double k3, double kp1, double kp2, double kp3) {
    double kk = k1 * k1 + k2 * k2 + k3 * k3;
    switch (kind) {
        case SYM_DX1: return I * kp1;          /* d/dx1 <-> i k'_1 */
        case SYM_DX2: return I * kp2;
        case SYM_DX3: return I * kp3;
        case SYM_LAP: return -kk;              /* Laplacian <-> -|k|^2 */
        case SYM_BIHARM: return kk * kk;       /* biharmonic <-> |k|^4  (Eq. 4) */
    }
    return 0;
}

static void to_complex(int64_t M, const double* f, cplx* a) {
    for (int64_t i = 0; i < M; ++i) a[i] = f[i];
}

/* out = Re F^{-1}[ sym(k) F f ]  (the spectral operator of kind `kind`; D3). */
void or_spectral_scalar(int n1, int n2, int n3, int kind, const double* f, double* out) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    cplx* a = (cplx*)malloc(sizeof(cplx) * (size_t)M);
    to_complex(M, f, a);
    or_fft3(n1, n2, n3, a, -1);
    for (int i3 = 0; i3 < n3; ++i3)
        for (int i2 = 0; i2 < n2; ++i2)
            for (int i1 = 0; i1 < n1; ++i1) {
                int64_t id = i1 + (int64_t)n1 * (i2 + (int64_t)n2 * i3);
                a[id] *= symbol(kind, wavenum(i1, n1), wavenum(i2, n2), wavenum(i3, n3),
                                wavenum_odd(i1, n1), wavenum_odd(i2, n2), wavenum_odd(i3, n3));
            }
    or_fft3(n1, n2, n3, a, +1);
    for (int64_t i = 0; i < M; ++i) out[i] = creal(a[i]) / (double)M;
    free(a);
}

/* grad f = (d1 f, d2 f, d3 f)  ("grad rho = (d1 rho, d2 rho, d3 rho)") */
void or_grad(int n1, int n2, int n3, const double* f, double* out3) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    for (int a = 0; a < 3; ++a) or_spectral_scalar(n1, n2, n3, SYM_DX1 + a, f, out3 + a * M);
}

/* div u = sum_a d_a u_a  (Eq. 2d; D3) */
void or_div(int n1, int n2, int n3, const double* u3, double* out) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    double* t = (double*)malloc(sizeof(double) * (size_t)M);
    memset(out, 0, sizeof(double) * (size_t)M);
    for (int a = 0; a < 3; ++a) {
        or_spectral_scalar(n1, n2, n3, SYM_DX1 + a, u3 + a * M, t);
        for (int64_t i = 0; i < M; ++i) out[i] += t[i];
    }
    free(t);
}

/* Regularisation operator, componentwise: out = beta * A u with a(k) = |k|^2 (reg=1, A = -Laplacian,
 * H1-seminorm) or |k|^4 (reg=2, A = biharmonic, Eq. 2a / P:L153 Eq. 4).  D3/D12, reading A4. */
void or_reg_apply(int n1, int n2, int n3, int reg, double beta, const double* u3, double* out3) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    cplx* a = (cplx*)malloc(sizeof(cplx) * (size_t)M);
    for (int c = 0; c < 3; ++c) {
        to_complex(M, u3 + c * M, a);
        or_fft3(n1, n2, n3, a, -1);
        for (int i3 = 0; i3 < n3; ++i3)
            for (int i2 = 0; i2 < n2; ++i2)
                for (int i1 = 0; i1 < n1; ++i1) {
                    double k1 = wavenum(i1, n1), k2 = wavenum(i2, n2), k3 = wavenum(i3, n3);
                    double kk = k1 * k1 + k2 * k2 + k3 * k3;
                    double ak = (reg == 1) ? kk : kk * kk;
                    a[i1 + (int64_t)n1 * (i2 + (int64_t)n2 * i3)] *= beta * ak;
                }
        or_fft3(n1, n2, n3, a, +1);
        for (int64_t i = 0; i < M; ++i) out3[c * M + i] = creal(a[i]) / (double)M;
    }
    free(a);
}

/* Leray projection L = I - grad Lap^{-1} div (Eq. 4): per mode,
 * L_hat(k) = I - k' k'^T / |k'|^2 for |k'| > 0, identity for k' = 0 (D3; readings A2, A3). */
static void leray_spectral(int n1, int n2, int n3, cplx* a0, cplx* a1, cplx* a2) {
    for (int i3 = 0; i3 < n3; ++i3)
        for (int i2 = 0; i2 < n2; ++i2)
            for (int i1 = 0; i1 < n1; ++i1) {
                int64_t id = i1 + (int64_t)n1 * (i2 + (int64_t)n2 * i3);
                double k1 = wavenum_odd(i1, n1), k2 = wavenum_odd(i2, n2), k3 = wavenum_odd(i3, n3);
                double kk = k1 * k1 + k2 * k2 + k3 * k3;
                if (kk == 0.0) continue;
                cplx kdot = k1 * a0[id] + k2 * a1[id] + k3 * a2[id];
                a0[id] -= k1 * kdot / kk;
                a1[id] -= k2 * kdot / kk;
                a2[id] -= k3 * kdot / kk;
            }
}

void or_leray(int n1, int n2, int n3, const double* u3, double* out3) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    cplx* a[3];
    for (int c = 0; c < 3; ++c) {
        a[c] = (cplx*)malloc(sizeof(cplx) * (size_t)M);
        to_complex(M, u3 + c * M, a[c]);
        or_fft3(n1, n2, n3, a[c], -1);
    }
    leray_spectral(n1, n2, n3, a[0], a[1], a[2]);
    for (int c = 0; c < 3; ++c) {
        or_fft3(n1, n2, n3, a[c], +1);
        for (int64_t i = 0; i < M; ++i) out3[c * M + i] = creal(a[c][i]) / (double)M;
        free(a[c]);
    }
}

/* Spectral preconditioner (§III-A: "the inverse of the biharmonic operator"), D13:
 * z = F^{-1}[ F r / (beta a_hat(k)) ], a_hat(0) = 1 (reading A5), followed by L when isochoric. */
void or_precond(int n1, int n2, int n3, int reg, double beta, int iso, const double* r3, double* z3) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    cplx* a[3];
    for (int c = 0; c < 3; ++c) {
        a[c] = (cplx*)malloc(sizeof(cplx) * (size_t)M);
        to_complex(M, r3 + c * M, a[c]);
        or_fft3(n1, n2, n3, a[c], -1);
        for (int i3 = 0; i3 < n3; ++i3)
            for (int i2 = 0; i2 < n2; ++i2)
                for (int i1 = 0; i1 < n1; ++i1) {
                    double k1 = wavenum(i1, n1), k2 = wavenum(i2, n2), k3 = wavenum(i3, n3);
                    double kk = k1 * k1 + k2 * k2 + k3 * k3;
                    double ak = (reg == 1) ? kk : kk * kk;
                    if (kk == 0.0) ak = 1.0;
                    a[c][i1 + (int64_t)n1 * (i2 + (int64_t)n2 * i3)] /= beta * ak;
                }
    }
    if (iso) leray_spectral(n1, n2, n3, a[0], a[1], a[2]);
    for (int c = 0; c < 3; ++c) {
        or_fft3(n1, n2, n3, a[c], +1);
        for (int64_t i = 0; i < M; ++i) z3[c * M + i] = creal(a[c][i]) / (double)M;
        free(a[c]);
    }
}

/* --------------------------------------------------------------------------------------------
 * Tricubic interpolation (§III-C2: "64 scalar values ... 64 coefficients (4^3)"),
 * D4, reading A6/A7: tensor-product cubic Lagrange on nodes q-1..q+2 with periodic wrap.
 * Points are given in CELL coordinates s (x = h*s).  q = floor(s), t = s - q in [0,1).
 * ------------------------------------------------------------------------------------------ */
static void lagrange_weights(double t, double w[4]) {
    w[0] = -t * (t - 1.0) * (t - 2.0) / 6.0;          /* node q-1 */
    w[1] = (t + 1.0) * (t - 1.0) * (t - 2.0) / 2.0;   /* node q   */
    w[2] = -(t + 1.0) * t * (t - 2.0) / 2.0;          /* node q+1 */
    w[3] = (t + 1.0) * t * (t - 1.0) / 6.0;           /* node q+2 */
}

static int64_t wrap(int64_t i, int N) {
    int64_t r = i % N;
    return r < 0 ? r + N : r;
}

static double interp_at(int n1, int n2, int n3, const double* f, double s1, double s2, double s3) {
    double q1 = floor(s1), q2 = floor(s2), q3 = floor(s3);
    double w1[4], w2[4], w3[4];
    lagrange_weights(s1 - q1, w1);
    lagrange_weights(s2 - q2, w2);
    lagrange_weights(s3 - q3, w3);
    double acc = 0.0;
    for (int c = 0; c < 4; ++c)
        for (int b = 0; b < 4; ++b)
            for (int a = 0; a < 4; ++a) {
                int64_t j1 = wrap((int64_t)q1 + a - 1, n1);
                int64_t j2 = wrap((int64_t)q2 + b - 1, n2);
                int64_t j3 = wrap((int64_t)q3 + c - 1, n3);
                acc += w1[a] * w2[b] * w3[c] * f[j1 + (int64_t)n1 * (j2 + (int64_t)n2 * j3)];
            }
    return acc;
}

/* out[p] = I[f](s_p) for arbitrary points s (s1, s2, s3 arrays of length npts). */
void or_interp(int n1, int n2, int n3, const double* f, int64_t npts,
               const double* s1, const double* s2, const double* s3, double* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npts; ++p) out[p] = interp_at(n1, n2, n3, f, s1[p], s2[p], s3[p]);
}

/* Semi-Lagrangian gather at the departure points of a displacement field d (cell units):
 * out_i = I[f](i - d_i)  (D5/D6: s_i = i - d_i). */
void or_sl_gather(int n1, int n2, int n3, const double* f, const double* d3, double* out) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    #pragma omp parallel for schedule(static)
    for (int64_t id = 0; id < M; ++id) {
        int64_t i1 = id % n1, i2 = (id / n1) % n2, i3 = id / ((int64_t)n1 * n2);
        out[id] = interp_at(n1, n2, n3, f, (double)i1 - d3[id], (double)i2 - d3[M + id],
                            (double)i3 - d3[2 * M + id]);
    }
}

/* RK2 departure points (Eq. 6, with v -> sigma*v; D5), in cell units:
 *   X*_i = x_i - dt*sigma*v(x_i)                -> s*_i = i - sigma*dt*v(x_i)/h
 *   X_i  = x_i - dt/2*sigma*(v(x_i) + v(X*_i))  -> d_i = sigma*dt/2*(v(x_i) + I[v](s*_i))/h,  s_i = i - d_i
 * v(X*) needs "three interpolations", one per component, with shared weights. */
void or_departure(int n1, int n2, int n3, int nt, int sigma, const double* v3, double* d3) {
    const int64_t M = (int64_t)n1 * n2 * n3;
    const double dt = 1.0 / (double)nt;
    const double h[3] = {2.0 * PI / n1, 2.0 * PI / n2, 2.0 * PI / n3};
    #pragma omp parallel for schedule(static)
    for (int64_t id = 0; id < M; ++id) {
        int64_t i1 = id % n1, i2 = (id / n1) % n2, i3 = id / ((int64_t)n1 * n2);
        double s1 = (double)i1 - sigma * dt * v3[id] / h[0];
        double s2 = (double)i2 - sigma * dt * v3[M + id] / h[1];
        double s3 = (double)i3 - sigma * dt * v3[2 * M + id] / h[2];
        for (int a = 0; a < 3; ++a) {
            double vstar = interp_at(n1, n2, n3, v3 + a * M, s1, s2, s3);
            d3[a * M + id] = sigma * 0.5 * dt * (v3[a * M + id] + vstar) / h[a];
        }
    }
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the OpenMP loops (bench.py's CPU-baseline protocol times 1 and nproc threads;
 * SURVEY §8(d)).  Execution control only: the arithmetic does not depend on it. */
void or_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
