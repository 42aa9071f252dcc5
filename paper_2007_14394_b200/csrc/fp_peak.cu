// fp_peak.cu — FMA-pipe throughput microbenchmark (roofline denominators for the
// FP-bound tracing kernels; MEASURED_PEAKS.json only carries HBM and bf16 GEMM).
// Every thread runs 8 independent FMA chains; the grid is 8 CTAs of 256 threads
// per SM, enough to saturate the pipes. Rate = FMA instructions per second.
#include <cuda_runtime.h>

namespace sdfgi_dev {

template <typename T>
__global__ void __launch_bounds__(256) k_fma_peak(T* out, int iters, T a, T b) {
    T x0 = threadIdx.x * T(1e-3), x1 = x0 + T(1), x2 = x0 + T(2), x3 = x0 + T(3);
    T x4 = x0 + T(4), x5 = x0 + T(5), x6 = x0 + T(6), x7 = x0 + T(7);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == T(-12345)) out[0] = s;  // keep the chains alive
}

double measure_fma_rate(bool f64, cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    void* out = nullptr;
    cudaMalloc(&out, 16);
    const int blocks = sms * 8, threads = 256;
    const int iters = f64 ? 512 : 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, st);
        if (f64)
            k_fma_peak<double><<<blocks, threads, 0, st>>>((double*)out, iters, 0.999999, 1e-7);
        else
            k_fma_peak<float><<<blocks, threads, 0, st>>>((float*)out, iters, 0.999f, 1e-4f);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    double fmas = double(blocks) * threads * iters * 16.0 * 8.0;
    return fmas / (best * 1e-3);
}

}  // namespace sdfgi_dev
