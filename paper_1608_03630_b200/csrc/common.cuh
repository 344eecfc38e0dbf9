// common.cuh -- shared device helpers of the B200 diffreg library (product path; no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dr {

template <typename T>
struct __align__(2 * sizeof(T)) Cx {
    T re, im;
};

template <typename T>
__host__ __device__ __forceinline__ Cx<T> cx(T r, T i) { Cx<T> c; c.re = r; c.im = i; return c; }
template <typename T>
__device__ __forceinline__ Cx<T> operator+(Cx<T> a, Cx<T> b) { return cx(a.re + b.re, a.im + b.im); }
template <typename T>
__device__ __forceinline__ Cx<T> operator-(Cx<T> a, Cx<T> b) { return cx(a.re - b.re, a.im - b.im); }
template <typename T>
__device__ __forceinline__ Cx<T> cmul(Cx<T> a, Cx<T> b) {
    return cx(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
template <typename T>
__device__ __forceinline__ Cx<T> conj(Cx<T> a) { return cx(a.re, -a.im); }
template <typename T>
__device__ __forceinline__ Cx<T> scale(Cx<T> a, T s) { return cx(a.re * s, a.im * s); }
// multiply by i*s
template <typename T>
__device__ __forceinline__ Cx<T> mul_i(Cx<T> a, T s) { return cx(-a.im * s, a.re * s); }

// Grid geometry: power-of-two extents, x1 fastest.
struct Grid {
    int n1, n2, n3;        // extents
    int l1, l2, l3;        // log2 extents
    int64_t M;             // n1*n2*n3
    int n1c;               // n1/2 + 1: half-spectrum row length
    int n1p;               // padded spectrum row stride (>= n1c, multiple of 16)
    int64_t S;             // n3*n2*n1p complex entries of one spectrum
};

__device__ __forceinline__ int wrapi(int i, int n) { return i & (n - 1); }  // n is a power of two

// Signed wavenumber of index i on an axis of length n: k in {-n/2+1, ..., n/2}.
__device__ __forceinline__ int wavenum(int i, int n) { return (i <= (n >> 1)) ? i : i - n; }
// First-order symbols zero the Nyquist mode (reading A2).
__device__ __forceinline__ int wavenum_odd(int i, int n) { return (i == (n >> 1)) ? 0 : wavenum(i, n); }

}  // namespace dr
