// HBM read-bandwidth probe: what a read-only stream can reach on this B200, next to
// MEASURED_PEAKS.json's copy figure (read + write).  The collision kernel (K2) is a
// read-only stream, so this is its practical ceiling.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/read_peak profiles/read_peak.cu
//   /tmp/read_peak    -> one JSON line per variant
//
// Variants over a 4 GiB buffer (>> 126 MB L2), best of 5 after warm-up, CUDA events:
//   ldg128      grid-stride 16-byte streaming loads (__ldcs), 8 in flight per thread, 4 x 148 x 512 threads
//   tma<B>      1-warp CTAs, 3-stage cp.async.bulk ring of B-byte chunks, 13 CTAs/SM
//               (the collision kernel's pipeline shape), chunks walked contiguously
//   tma512x8    as tma but each stage = 8 chunks of 512 B spaced 14 KB apart (the packed
//               history's plane pattern at s ~ 900)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void ldg128(const double2* __restrict__ p, size_t n4, double* out) {
    double acc = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n4; i += 8 * stride) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    for (; i < n4; i += stride) { double2 v = __ldcs(p + i); acc += v.x + v.y; }
    if (acc == 1.2345) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CHUNKS>
__global__ void __launch_bounds__(32) tma_ring(const char* base, size_t chunk_bytes, size_t nstage_total,
                                                size_t spacing, unsigned* next, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = (uint64_t*)(sm + 3 * CHUNKS * chunk_bytes);
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    double acc = 0.0;
    unsigned g = 0;
    const size_t per_task = 32;   // stages per task (like 32 slices)
    const size_t ntask = nstage_total / per_task;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(next, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntask) break;
        auto issue = [&](size_t stage, unsigned slot) {
            const uint32_t bytes = (uint32_t)(CHUNKS * chunk_bytes);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[slot])), "r"(bytes) : "memory");
            for (int c = 0; c < CHUNKS; ++c) {
                const char* src = base + (stage * CHUNKS + c) * (CHUNKS > 1 ? spacing : chunk_bytes);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(sm + (slot * CHUNKS + c) * chunk_bytes)), "l"(src), "r"((uint32_t)chunk_bytes),
                             "r"(su32(&bar[slot])) : "memory");
            }
        };
        const size_t s0 = (size_t)t * per_task;
        if (lane == 0)
            for (int i = 0; i < 3; ++i) issue(s0 + i, (g + i) % 3);
        for (size_t i = 0; i < per_task; ++i, ++g) {
            const unsigned slot = g % 3, par = (g / 3) & 1;
            asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}"
                         ::"r"(su32(&bar[slot])), "r"(par) : "memory");
            const double* d = (const double*)(sm + slot * CHUNKS * chunk_bytes);
            for (size_t k = lane; k < CHUNKS * chunk_bytes / 8; k += 32) acc += d[k];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0 && i + 3 < per_task) issue(s0 + i + 3, slot);
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    const size_t bytes = (size_t)4 << 30;
    char* buf;
    double* out;
    unsigned* next;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&out, 8);
    cudaMalloc(&next, 4);
    cudaMemset(buf, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto best = [&](auto fn, size_t moved) {
        float bm = 1e30f;
        for (int r = 0; r < 7; ++r) {
            cudaMemset(next, 0, 4);
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 2 && ms < bm) bm = ms;
        }
        return moved / (bm * 1e-3) / 1e9;
    };
    {
        const size_t n4 = bytes / 16;
        double gbs = best([&] { ldg128<<<4 * sms, 512>>>((const double2*)buf, n4, out); }, bytes);
        printf("{\"variant\": \"ldg128\", \"gbs\": %.1f}\n", gbs);
    }
    for (size_t cb : {4096, 8192}) {
        const size_t smem = 3 * cb + 64;
        cudaFuncSetAttribute(tma_ring<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_ring<1>, 32, smem);
        if (occ > 13) occ = 13;
        const size_t nst = bytes / cb;
        double gbs = best([&] { tma_ring<1><<<sms * occ, 32, smem>>>(buf, cb, nst, cb, next, out); }, nst * cb);
        printf("{\"variant\": \"tma%zu\", \"ctas_per_sm\": %d, \"gbs\": %.1f}\n", cb, occ, gbs);
    }
    {
        // 8 x 512 B per stage, chunks 14 KB apart, stages walking with 4 KB offsets inside a 14 KB x 8 frame
        const size_t cb = 512, spacing = 14336;
        const size_t smem = 3 * 8 * cb + 64;
        cudaFuncSetAttribute(tma_ring<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_ring<8>, 32, smem);
        if (occ > 13) occ = 13;
        const size_t nst = (bytes - 8 * spacing) / (8 * spacing) * (spacing / cb) / 8;   // keeps addresses in range
        double gbs = best([&] { tma_ring<8><<<sms * occ, 32, smem>>>(buf, cb, nst, cb, next, out); }, nst * 8 * cb);
        printf("{\"variant\": \"tma512x8_contig\", \"ctas_per_sm\": %d, \"gbs\": %.1f}\n", occ, gbs);
        (void)spacing;
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
