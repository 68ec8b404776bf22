// Microbenchmark: latency per element of the fold's float64 chain on one warp
// (lane = dimension), data resident in shared memory.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void chain(const float *g, int n, double *out, long long *cyc) {
    __shared__ float buf[128 * 32];
    __shared__ unsigned char flag[128];
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) buf[i] = g[i];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) flag[i] = (i % 7 == 3) ? 2 : 0;
    __syncthreads();
    const int lane = threadIdx.x;
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < n; it++) {
#pragma unroll 8
        for (int r = 0; r < 128; r++) {
            const double v = (double)buf[r * 32 + lane];
            if (MODE == 0) {
                acc = __dadd_rn(acc, v);
            } else if (MODE == 1) {
                const unsigned char fl = flag[r];
                const double add = __dadd_rn(acc, v);
                acc = fl == 1 ? v : (fl == 0 ? add : acc);
            } else {
                const unsigned char fl = flag[r];
                const double vv = fl == 0 ? v : 0.0;  // skip -> add exact zero? (not exact for -0.0)
                acc = __dadd_rn(acc, vv);
            }
        }
    }
    long long t1 = clock64();
    out[lane] = acc;
    if (lane == 0) *cyc = t1 - t0;
}

int main() {
    float *g;
    double *o;
    long long *c, h;
    cudaMalloc(&g, 128 * 32 * 4);
    cudaMemset(g, 0, 128 * 32 * 4);
    cudaMalloc(&o, 32 * 8);
    cudaMalloc(&c, 8);
    const int n = 100;
    chain<0><<<1, 32>>>(g, n, o, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("plain dadd chain: %.2f cycles/elem\n", (double)h / (n * 128));
    chain<1><<<1, 32>>>(g, n, o, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dadd + flag selects: %.2f cycles/elem\n", (double)h / (n * 128));
    chain<2><<<1, 32>>>(g, n, o, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dadd of masked value: %.2f cycles/elem\n", (double)h / (n * 128));
    return 0;
}
