// Microbenchmark: throughput of warp shuffles vs shared-memory loads (does SHFL share the LDS datapath?)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
    __shared__ float s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = (float)i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float a0 = lane, a1 = lane + 1, a2 = lane + 2, a3 = lane + 3, acc = 0.f;
    int base = lane + (threadIdx.x >> 5) * 64;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // 4 independent LDS
            const int c = (base + it * 8) & 1023;
            acc += s[c] + s[c + 1] + s[c + 2] + s[c + 3];
        } else if (MODE == 1) {  // 4 independent SHFL
            a0 = __shfl_sync(0xffffffffu, a0, (lane + 1) & 31);
            a1 = __shfl_sync(0xffffffffu, a1, (lane + 2) & 31);
            a2 = __shfl_sync(0xffffffffu, a2, (lane + 3) & 31);
            a3 = __shfl_sync(0xffffffffu, a3, (lane + 5) & 31);
        } else {  // 2 LDS + 2 SHFL interleaved
            const int c = (base + it * 8) & 1023;
            acc += s[c] + s[c + 1];
            a0 = __shfl_sync(0xffffffffu, a0, (lane + 1) & 31);
            a1 = __shfl_sync(0xffffffffu, a1, (lane + 2) & 31);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + a0 + a1 + a2 + a3;
}

int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 8192;
    const char* names[3] = {"4 LDS", "4 SHFL", "2 LDS + 2 SHFL"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(o, iters);
            if (mode == 1) k<1><<<148 * 8, 256>>>(o, iters);
            if (mode == 2) k<2><<<148 * 8, 256>>>(o, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double warp_iters = 148.0 * 8 * 8 * iters;
            if (rep) printf("%-16s %.3f ms, %.2f SM-cycles per warp-iteration (4 ops) at 1.9 GHz\n", names[mode], ms,
                            ms * 1e-3 * 1.9e9 * 148 / warp_iters);
        }
    }
    return 0;
}
