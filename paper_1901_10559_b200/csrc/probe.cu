// Measurement probe: sustained fp64 FMA throughput of this GPU, the second
// roof (next to HBM bandwidth) of the TensorSketch kernel's FFT work.
// Diagnostic only -- nothing on the sketch / ID path calls it.
#include "common.cuh"

namespace {

constexpr int kChains = 8;  // independent DFMA chains per thread (hide the pipe latency)

__global__ void __launch_bounds__(256) dfma_kernel(int iters, double seed, double* sink) {
    double a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
    const double m = 0.999999999, b = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = fma(a[c], m, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += a[c];
    if (s == 12345.678) sink[0] = s;  // never true; keeps the chains live
}

}  // namespace

extern "C" double ids_probe_fp64_tflops(void* stream) {
    cudaStream_t st = as_stream(stream);
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return -1.0;
    double* sink = nullptr;
    if (cudaMallocAsync(&sink, sizeof(double), st) != cudaSuccess) return -1.0;
    const int threads = 256, blocks = sms * 8, iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_kernel<<<blocks, threads, 0, st>>>(iters / 8, 1.0, sink);  // warm-up
    ids_count_launch();
    cudaEventRecord(e0, st);
    dfma_kernel<<<blocks, threads, 0, st>>>(iters, 1.0, sink);
    ids_count_launch();
    cudaEventRecord(e1, st);
    float ms = 0.f;
    double out = -1.0;
    if (cudaEventSynchronize(e1) == cudaSuccess && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess &&
        ms > 0.f)
        out = 2.0 * kChains * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(sink, st);
    cudaGetLastError();
    return out;
}
