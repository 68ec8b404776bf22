// Microbenchmark: cost of alternating kernels with different shared-memory
// footprints (SM carveout reconfiguration) on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_small(float *x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.f; }
__global__ void k_big(float *x) {
    extern __shared__ float sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) x[1] += sm[5];
}
int main() {
    float *x;
    cudaMalloc(&x, 64);
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 4; mode++) {
        if (mode == 2) {
            cudaFuncSetAttribute(k_small, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            cudaFuncSetAttribute(k_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        }
        for (int w = 0; w < 2; w++) {
            cudaEventRecord(a);
            for (int i = 0; i < 200; i++) {
                if (mode == 0 || mode == 2 || mode == 3) k_small<<<148, 128>>>(x);
                if (mode != 3) k_big<<<128, 128, 192 * 1024>>>(x);
                else k_big<<<128, 128, 1024>>>(x);
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const char *names[] = {"small+big(192K)", "big only", "small+big, carveout 100", "small+big(1K)"};
        printf("%-28s %.2f us per iteration\n", names[mode], ms * 1e3 / 200);
    }
    return 0;
}
