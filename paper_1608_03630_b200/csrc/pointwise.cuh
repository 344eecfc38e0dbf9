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

// lambda(1) = rho_R - rho(1)   (Eq. 3)
template <typename T>
__global__ void k_sub(int64_t M, const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}

template <typename T>
__global__ void k_scale(int64_t M, const T* __restrict__ a, T* __restrict__ out, T s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = s * a[i];
}

// b~ = dt sum_j w_j lambda~_j G_j, w_0 = w_nt = 1/2 (trapezoid, reading A12).
// lambda~_j (j < nt) are consecutive scalar slices at lt; lambda~_nt = sgn_last * last.
// G_j: consecutive vector slices at G (stride 3M).
template <typename T>
__global__ void k_quadrature(int64_t M, int nt, const T* __restrict__ lt, const T* __restrict__ last, T sgn_last,
                             const T* __restrict__ G, T* __restrict__ b, T dt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        T b0 = T(0), b1 = T(0), b2 = T(0);
        for (int j = 0; j <= nt; ++j) {
            const T w = (j == 0 || j == nt) ? T(0.5) * dt : dt;
            const T l = w * ((j < nt) ? lt[(int64_t)j * M + i] : sgn_last * last[i]);
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

}  // namespace dr
