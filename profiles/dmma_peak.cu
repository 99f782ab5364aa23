// FP64 tensor-core (DMMA) peak probe, beside fp64_peak.cu (DFMA): the two FP64
// ceilings a Sigma kernel can be held against on this B200.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_peak profiles/dmma_peak.cu
//   /tmp/dmma_peak            -> one JSON line {"dmma_tflops": ..., ...}
//
// mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 (SASS DMMA.8x8x4): 8x8x4 = 256 FMA =
// 512 flop per warp instruction.  CH independent accumulator chains per warp (the
// DMMA latency is hidden by the chains and by the warps per SM), timed with CUDA
// events after a warm-up, for several warps-per-SM / chain counts; the best is the peak.
#include <cuda_runtime.h>
#include <stdio.h>

template <int CH>
__global__ void dmma_chains(double* out, int iters) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-9, b = 0.999999 - lane * 1e-9;
    double c[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) { c[i][0] = i * 1e-3; c[i][1] = -i * 1e-3; }
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < CH; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;   // keep the chains live
}

template <int CH>
static double run(int sms, int warps_per_cta, int ctas_per_sm, int iters, double* out, float* ms_out) {
    const int threads = 32 * warps_per_cta, blocks = sms * ctas_per_sm;
    dmma_chains<CH><<<blocks, threads>>>(out, 100);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dmma_chains<CH><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    *ms_out = best;
    const double flops = 512.0 * CH * iters * (double)(threads / 32) * blocks;
    return flops / (best * 1e-3) / 1e12;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    double best = 0.0;
    float best_ms = 0.f;
    int best_w = 0, best_ch = 0;
    const int warps[] = {4, 8, 16};
    for (int w : warps) {
        float ms = 0.f;
        double t = run<4>(sms, w, 2, 4000, out, &ms);
        printf("{\"probe\": \"dmma\", \"chains\": 4, \"warps_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", 2 * w, t, ms);
        if (t > best) { best = t; best_ms = ms; best_w = 2 * w; best_ch = 4; }
        t = run<8>(sms, w, 2, 2000, out, &ms);
        printf("{\"probe\": \"dmma\", \"chains\": 8, \"warps_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", 2 * w, t, ms);
        if (t > best) { best = t; best_ms = ms; best_w = 2 * w; best_ch = 8; }
    }
    printf("{\"dmma_tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, \"kernel_ms\": %.3f, "
           "\"method\": \"mma.sync m8n8k4 f64, %d independent chains/warp, %d warps/SM, best of 5 per point\"}\n",
           best, sms, clk / 1000, best_ms, best_ch, best_w);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
