// Launch-latency probe for the step sequencing choices:
//   host      K dependent launches of a 1924 x 32 no-op kernel from the host, PDL on
//   host_nopdl the same without programmatic stream serialization
//   tail      a device-driven chain: each grid's last CTA tail-launches the next grid
//             (CDP2 cudaStreamTailLaunch), the host launches only the first
//   barrier   one persistent grid (148 x 4 CTAs) crossing K software grid barriers
// Reported: microseconds per dependent step.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=true -o /tmp/ll profiles/launch_latency.cu -lcudadevrt
#include <cuda_runtime.h>
#include <stdio.h>

__device__ unsigned g_done;
__device__ volatile unsigned g_gen;
__device__ unsigned g_count;

__global__ void noop_pdl(int* flag) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (flag[0] == 12345) flag[1] = 1;
}

__global__ void chain(int* flag, int left) {
    if (flag[0] == 12345) flag[1] = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&g_done, 1u) == gridDim.x - 1) {
            g_done = 0;
            if (left > 1) chain<<<gridDim.x, blockDim.x, 0, cudaStreamTailLaunch>>>(flag, left - 1);
        }
    }
}

__device__ void grid_barrier(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = g_gen;
        __threadfence();
        if (atomicAdd(&g_count, 1u) == nblocks - 1) {
            g_count = 0;
            __threadfence();
            g_gen = gen + 1;
        } else {
            while (g_gen == gen) { __nanosleep(32); }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void barriers(int* flag, int k) {
    for (int i = 0; i < k; ++i) {
        if (flag[0] == 12345) flag[1] = i;
        grid_barrier(gridDim.x);
    }
}

int main() {
    int* flag;
    cudaMalloc(&flag, 8);
    cudaMemset(flag, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int K = 2000;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float ms;
    for (int pdl = 1; pdl >= 0; --pdl) {
        for (int grid : {1924, 148}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(32);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl;
            for (int r = 0; r < 2; ++r) {
                cudaEventRecord(e0);
                for (int i = 0; i < K; ++i) cudaLaunchKernelEx(&cfg, noop_pdl, flag);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"mode\": \"%s\", \"grid\": %d, \"us_per_step\": %.3f}\n", pdl ? "host_pdl" : "host_nopdl", grid,
                   1e3 * ms / K);
        }
    }
    for (int grid : {1924, 148}) {
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            chain<<<grid, 32>>>(flag, K);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"mode\": \"tail\", \"grid\": %d, \"us_per_step\": %.3f, \"err\": \"%s\"}\n", grid, 1e3 * ms / K,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int per : {1, 4}) {
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            barriers<<<sms * per, 128>>>(flag, K);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"mode\": \"barrier\", \"grid\": %d, \"us_per_step\": %.3f, \"err\": \"%s\"}\n", sms * per,
               1e3 * ms / K, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
