// Green-context probe: split the SMs into groups, make a stream per group,
// launch runtime-API kernels on it over memory from cudaMalloc/cudaMallocAsync
// (primary context), and report the SM ids each group's CTAs ran on.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>
#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char *s; cuGetErrorString(r_, &s); printf("%s failed: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)
__global__ void k_smid(int *out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned sm; asm("mov.u32 %0, %%smid;" : "=r"(sm));
    if (threadIdx.x == 0) out[blockIdx.x] = sm;
    for (int k = 0; k < 100000 && i < n; k++) __nanosleep(10);
}
int main() {
    RK(cudaSetDevice(0));
    RK(cudaFree(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("SMs: %u\n", all.sm.smCount);
    unsigned ng = 8; CUdevResource groups[8]; CUdevResource rem;
    CK(cuDevSmResourceSplitByCount(groups, &ng, &all, &rem, 0, 16));
    printf("groups %u of %u SMs, remaining %u\n", ng, groups[0].sm.smCount, rem.sm.smCount);
    std::vector<cudaStream_t> st(ng);
    for (unsigned g = 0; g < ng; g++) {
        CUdevResourceDesc d; CK(cuDevResourceGenerateDesc(&d, &groups[g], 1));
        CUgreenCtx gc; CK(cuGreenCtxCreate(&gc, d, dev, CU_GREEN_CTX_DEFAULT_STREAM));
        CUstream s; CK(cuGreenCtxStreamCreate(&s, gc, CU_STREAM_NON_BLOCKING, 0));
        st[g] = (cudaStream_t)s;
    }
    int *out; RK(cudaMalloc(&out, 8 * 64 * sizeof(int)));
    int *out2; RK(cudaMallocAsync(&out2, 64 * sizeof(int), st[0]));
    for (unsigned g = 0; g < ng; g++) k_smid<<<64, 32, 0, st[g]>>>(out + g * 64, 0);
    k_smid<<<64, 32, 0, st[0]>>>(out2, 0);
    RK(cudaGetLastError());
    RK(cudaDeviceSynchronize());
    std::vector<int> h(8 * 64);
    RK(cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost));
    for (unsigned g = 0; g < ng; g++) {
        int mn = 1 << 30, mx = -1;
        for (int b = 0; b < 64; b++) { mn = std::min(mn, h[g * 64 + b]); mx = std::max(mx, h[g * 64 + b]); }
        std::vector<int> seen(256, 0); int nd = 0;
        for (int b = 0; b < 64; b++) if (!seen[h[g * 64 + b]]++) nd++;
        printf("group %u: CTAs on %d distinct SMs (ids %d..%d)\n", g, nd, mn, mx);
    }
    printf("ok\n");
    return 0;
}
