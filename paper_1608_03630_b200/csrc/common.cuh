// common.cuh -- shared device helpers of the B200 diffreg library (product path; no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// DR_CHECK builds (DR_CHECK=1 python paper_1608_03630_b200/build.py -> libdiffreg_check.so) turn on
// device-side bounds checks of every computed shared-memory and ghosted-field index.
#ifdef DR_CHECK
#include <cassert>
#define DR_ASSERT(c) assert(c)
#else
#define DR_ASSERT(c) ((void)0)
#endif

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

// Grid geometry of one rank's slab: power-of-two extents, x1 fastest.  With one rank the slab is the
// whole grid.  With P ranks rank r owns the x3 planes [z0, z0 + n3) of the global
// n3g, and the scalar fields that semi-Lagrangian gathers read carry zg ghost planes below and zgh
// above (ghost = 1: x3 indices of gathers are slab-local with ghosts instead of periodic wraps).
struct Grid {
    int n1, n2, n3;        // local extents (n3 = slab thickness)
    int l1, l2, l3;        // log2 extents
    int64_t M;             // n1*n2*n3 local voxels
    int n1c;               // n1/2 + 1: half-spectrum row length
    int n1p;               // padded spectrum row stride (>= n1c, multiple of 16)
    int64_t S;             // n3*n2*n1p complex entries of one local spectrum
    int z0, n3g;           // global x3 offset of the slab, global x3 extent
    int zg, zgh;           // ghost planes below / above the slab (0 with one rank)
    int ghost;             // 1: slab mode (gathers index x3 through the ghosts, no wrap)
};

__device__ __forceinline__ int wrapi(int i, int n) { return i & (n - 1); }  // n is a power of two
// extents that are not powers of two (Bluestein passes, one rank): a remainder then
__device__ __forceinline__ int wrap2(int i, int n) { return (n & (n - 1)) ? ((i % n) + n) % n : (i & (n - 1)); }

// Signed wavenumber of index i on an axis of length n: k in {-n/2+1, ..., n/2}.
__device__ __forceinline__ int wavenum(int i, int n) { return (i <= (n >> 1)) ? i : i - n; }
// First-order symbols zero the Nyquist mode (reading A2).
__device__ __forceinline__ int wavenum_odd(int i, int n) { return (i == (n >> 1)) ? 0 : wavenum(i, n); }

}  // namespace dr
