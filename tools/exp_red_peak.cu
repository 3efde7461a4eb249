// Peak rate of scattered fp64 / u64 reductions into an L2-resident buffer
// (the bound of the streaming CSR sketch).  Addresses from a multiplicative
// hash, no loads.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/exp_red_peak.cu -o tools/exp_red_peak.bin
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <class T>
__global__ void red_kernel(T* __restrict__ y, uint32_t mask, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t h = (uint32_t)i * 2654435761u;
        atomicAdd(y + ((h ^ (h >> 15)) & mask), (T)1);
    }
}

int main() {
    const int64_t n = 100000000;
    double* y;
    cudaMalloc(&y, 64 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int bits : {18, 21, 22}) {
        for (int g : {148 * 8, 148 * 16, 148 * 32}) {
            for (int kind = 0; kind < 2; ++kind) {
                float best = 1e9;
                for (int r = 0; r < 4; ++r) {
                    cudaEventRecord(e0);
                    if (kind == 0) red_kernel<double><<<g, 256>>>(y, (1u << bits) - 1, n);
                    else red_kernel<unsigned long long><<<g, 256>>>((unsigned long long*)y, (1u << bits) - 1, n);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (r && ms < best) best = ms;
                }
                printf("%s Y=%6d KB grid=%5d: %.3f ms  %.1f G red/s\n", kind ? "u64" : "f64",
                       (8 << bits) >> 10, g, best, n / best / 1e6);
            }
        }
    }
    return 0;
}
