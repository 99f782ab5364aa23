// FP64 FMA peak probe: the denominator of the Sigma kernel's FP64 roofline.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak profiles/fp64_peak.cu
//   /tmp/fp64_peak            -> one JSON line {"fp64_tflops": ..., "sms": ..., ...}
//
// 16 independent DFMA chains per thread, 8 warps x 4 CTAs per SM, timed with CUDA
// events after a warm-up.  MEASURED_PEAKS.json carries HBM and bf16 only, so this
// is the measured FP64 number the bench reports against.
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void fma_chains(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;   // keep the chains live
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    const int threads = 256, blocks = sms * 4, iters = 20000;
    fma_chains<<<blocks, threads>>>(out, 1000, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        fma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 16.0 * iters * (double)threads * blocks;
    printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, \"kernel_ms\": %.3f, "
           "\"method\": \"16 independent DFMA chains/thread, %d CTAs x %d threads, best of 5\"}\n",
           flops / (best * 1e-3) / 1e12, sms, clk / 1000, best, blocks, threads);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
