// Microbenchmark: shared-memory wavefronts of LDS.32 / LDS.64 / LDS.128 when lanes of a warp read
// overlapping consecutive words (the semi-Lagrangian stencil pattern: lane l reads around word l + c).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int c, int iters) {
    __shared__ __align__(16) float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (float)i;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float acc = 0.f;
    int base = (lane + c + w * 64) & 2047;
    for (int it = 0; it < iters; ++it) {
        const int col = (base + it * 16) & 2047;
        if (MODE == 0) {  // 4 x LDS.32 at col .. col+3
            acc += s[col] + s[col + 1] * 1.1f + s[col + 2] * 1.2f + s[col + 3] * 1.3f;
        } else if (MODE == 1) {  // 2 x LDS.128 at the 16-byte block containing col and the next one
            const int a = col & ~3;
            const float4 u = *reinterpret_cast<const float4*>(s + a);
            const float4 v = *reinterpret_cast<const float4*>(s + a + 4);
            acc += u.x + u.y * 1.1f + u.z * 1.2f + u.w * 1.3f + v.x * 1.4f + v.y * 1.5f + v.z * 1.6f + v.w * 1.7f;
        } else {  // 3 x LDS.64
            const int a = col & ~1;
            const float2 u = *reinterpret_cast<const float2*>(s + a);
            const float2 v = *reinterpret_cast<const float2*>(s + a + 2);
            const float2 x = *reinterpret_cast<const float2*>(s + a + 4);
            acc += u.x + u.y * 1.1f + v.x * 1.2f + v.y * 1.3f + x.x * 1.4f + x.y * 1.5f;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(o, 3, iters);
            if (mode == 1) k<1><<<148 * 8, 256>>>(o, 3, iters);
            if (mode == 2) k<2><<<148 * 8, 256>>>(o, 3, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double warp_iters = 148.0 * 8 * 8 * iters;
            if (rep) printf("mode %d: %.3f ms, %.2f SM-cycles per warp-iteration (at 1.9 GHz)\n", mode, ms,
                            ms * 1e-3 * 1.9e9 * 148 / warp_iters);
        }
    }
    return 0;
}
