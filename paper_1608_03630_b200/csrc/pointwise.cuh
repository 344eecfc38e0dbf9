// pointwise.cuh -- streaming kernels of the matvec that touch each voxel once (no stencil):
// incremental-state source at t_0, adjoint final condition, and the b~ time quadrature.
#pragma once
#include "common.cuh"

namespace dr {

// g_0 = rho~_0 + dt/2 f_0 = -(dt/2) vt . G_0   (Algorithm 2 with rho~(0) = 0, Eq. 5b; merged gather)
template <typename T>
__global__ void k_inc_init(int64_t M, const T* __restrict__ vt, const T* __restrict__ G0, T* __restrict__ g0, T c) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const T f = vt[i] * G0[i] + vt[M + i] * G0[M + i] + vt[2 * M + i] * G0[2 * M + i];
        g0[i] = -c * f;
    }
}

// DR_CHECK_FINITE: *flag = 1.0 if any of the n values is NaN or infinite (the input check of the
// main-path calls, SURVEY §8(b) DR_ERR_NONFINITE)
template <typename T>
__global__ void k_nonfinite(int64_t n, const T* __restrict__ x, double* __restrict__ flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1.0;
}

// lambda(1) = rho_R - rho(1)   (Eq. 3)
template <typename T>
__global__ void k_sub(int64_t M, const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}

// y = a x + b y (vector updates of the PCG iteration; coefficients in fp64, fields in T).  b == 0
// overwrites y without reading it (it may hold anything, NaN included).
template <typename T>
__global__ void k_axpby(int64_t n, double a, const T* __restrict__ x, double b, T* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = (b == 0.0) ? (T)(a * (double)x[i]) : (T)(a * (double)x[i] + b * (double)y[i]);
}

// NEXT-3 helpers.  rho~_j from the merged inc-state variable g_j = rho~_j + dt/2 f_j, f_j = -vt.G_j:
// rt = g + c vt.G_j (c = dt/2).
template <typename T>
__global__ void k_rt_from_g(int64_t M, const T* __restrict__ gj, const T* __restrict__ vt, const T* __restrict__ Gj,
                            T c, T* __restrict__ rt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        rt[i] = gj[i] + c * (vt[i] * Gj[i] + vt[M + i] * Gj[M + i] + vt[2 * M + i] * Gj[2 * M + i]);
}
// out (3 components) = lam * vt, the flux whose divergence is the source s = div(lam vt) of Eq. 5c
template <typename T>
__global__ void k_lam_vt(int64_t M, const T* __restrict__ lam, const T* __restrict__ vt, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const T l = lam[i];
        out[i] = l * vt[i];
        out[M + i] = l * vt[M + i];
        out[2 * M + i] = l * vt[2 * M + i];
    }
}
// b (3 components) (=|+=) w lam * grad  (the int lam grad rho~ dt term of b~, trapezoid weight w)
template <typename T>
__global__ void k_acc_lam_grad(int64_t M, const T* __restrict__ lam, const T* __restrict__ gr, T w,
                               T* __restrict__ b, int init) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const T l = w * lam[i];
#pragma unroll
        for (int a = 0; a < 3; ++a) b[a * M + i] = (init ? T(0) : b[a * M + i]) + l * gr[a * M + i];
    }
}

// det(I + grad u) pointwise from the nine derivatives d[a][b] = du_a/dx_b (Fig. 7 caption)
template <typename T>
__global__ void k_det(int64_t M, const T* __restrict__ d0, const T* __restrict__ d1, const T* __restrict__ d2,
                      T* __restrict__ det) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const double a00 = 1.0 + (double)d0[i], a01 = d0[M + i], a02 = d0[2 * M + i];
        const double a10 = d1[i], a11 = 1.0 + (double)d1[M + i], a12 = d1[2 * M + i];
        const double a20 = d2[i], a21 = d2[M + i], a22 = 1.0 + (double)d2[2 * M + i];
        det[i] = (T)(a00 * (a11 * a22 - a12 * a21) - a01 * (a10 * a22 - a12 * a20) + a02 * (a10 * a21 - a11 * a20));
    }
}

// min / max partials of a field (block b writes part[2b], part[2b+1]); k_minmax_final folds them
template <typename T>
__global__ void __launch_bounds__(256) k_minmax_parts(int64_t M, const T* __restrict__ a, double* __restrict__ part) {
    __shared__ double lo[256], hi[256];
    double l = 1e308, h = -1e308;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = (double)a[i];
        l = x < l ? x : l;
        h = x > h ? x : h;
    }
    lo[threadIdx.x] = l;
    hi[threadIdx.x] = h;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            lo[threadIdx.x] = fmin(lo[threadIdx.x], lo[threadIdx.x + s]);
            hi[threadIdx.x] = fmax(hi[threadIdx.x], hi[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = lo[0];
        part[2 * blockIdx.x + 1] = hi[0];
    }
}
__global__ void __launch_bounds__(256) k_minmax_final(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double lo[256], hi[256];
    double l = 1e308, h = -1e308;
    for (int i = threadIdx.x; i < n; i += 256) {
        l = fmin(l, part[2 * i]);
        h = fmax(h, part[2 * i + 1]);
    }
    lo[threadIdx.x] = l;
    hi[threadIdx.x] = h;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            lo[threadIdx.x] = fmin(lo[threadIdx.x], lo[threadIdx.x + s]);
            hi[threadIdx.x] = fmax(hi[threadIdx.x], hi[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = lo[0];
        out[1] = hi[0];
    }
}

// Device-scalar variants for the graph-captured PCG iteration: y = a x + b y with
// a = sa * (*pa or 1), b = (*pb or cb); scalars read once per thread.
template <typename T>
__global__ void k_axpby_dev(int64_t n, const double* __restrict__ pa, double sa, const T* __restrict__ x,
                            const double* __restrict__ pb, double cb, T* __restrict__ y) {
    const double a = pa ? sa * *pa : sa;
    const double b = pb ? *pb : cb;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = (T)(a * (double)x[i] + b * (double)y[i]);
}
// s[out] = s[num] / s[den]; with `shift`, also s[den] = s[num] (rz <- rz_new)
__global__ void k_scalar_ratio(double* s, int num, int den, int out, int shift) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const double v = s[num] / s[den];
        if (shift) s[den] = s[num];
        s[out] = v;
    }
}

template <typename T>
__global__ void k_scale(int64_t M, const T* __restrict__ a, T* __restrict__ out, T s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = s * a[i];
}

// b = dt sum_j w_j lambda_j G_j, w_0 = w_nt = 1/2 (trapezoid, reading A12; Eq. 4 with the
// time integral of P:L157).  lambda_j: slices lam + j * lstride; G_j: consecutive vector slices (3M).
template <typename T>
__global__ void k_quadrature(int64_t M, int nt, const T* __restrict__ lam, size_t lstride, const T* __restrict__ G,
                             T* __restrict__ b, T dt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        T b0 = T(0), b1 = T(0), b2 = T(0);
        for (int j = 0; j <= nt; ++j) {
            const T w = (j == 0 || j == nt) ? T(0.5) * dt : dt;
            const T l = w * lam[(size_t)j * lstride + i];
            const T* Gj = G + (int64_t)j * 3 * M;
            b0 += l * Gj[i];
            b1 += l * Gj[M + i];
            b2 += l * Gj[2 * M + i];
        }
        b[i] = b0;
        b[M + i] = b1;
        b[2 * M + i] = b2;
    }
}

// Deterministic fp64 dot product, pass 1: block b writes sum_{i in its grid-stride set} a_i c_i (and, with
// a2/c2, + the same for a second pair) to part[b].  Pass 2 (k_sum_parts, one block) adds the parts in
// block order.  Used by the objective (Eq. 2a) -- the inner product of S:L53, h^3 sum.
template <typename T>
__global__ void __launch_bounds__(256) k_dot_parts(int64_t M, const T* __restrict__ a, const T* __restrict__ c,
                                                   const T* __restrict__ a2, T* dummy, double* __restrict__ part,
                                                   int mode) {
    // mode 0: sum a*c; mode 1: sum (a - a2)^2
    __shared__ double red[256];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        if (mode == 0) acc += (double)a[i] * (double)c[i];
        else {
            const double d = (double)a[i] - (double)a2[i];
            acc += d * d;
        }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
    (void)dummy;
}

__global__ void __launch_bounds__(256) k_sum_parts(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double red[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) acc += part[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

}  // namespace dr
