// Probe: TMA tile::gather4 with a SWIZZLE_128B tensor map over an fp32 row
// matrix -- which box height the driver accepts and where the 4 rows land in
// shared memory.  nvcc -gencode arch=compute_100a,code=sm_100a -o tma_gather4 tma_gather4.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int col, int r0, int r1, int r2, int r3, float *out) {
    __shared__ __align__(1024) float buf[4 * 32];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf), bb = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bb), "r"(512));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3, %4, %5, %6}], [%7];\n" ::"r"(sb),
            "l"(&tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bb)
            : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(bb));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 128; i += blockDim.x) out[i] = buf[i];
}

int main() {
    const int R = 64, C = 64;
    std::vector<float> h(R * C);
    for (int r = 0; r < R; r++)
        for (int c = 0; c < C; c++) h[r * C + c] = r * 1000 + c;
    float *d, *o;
    cudaMalloc(&d, sizeof(float) * R * C);
    cudaMalloc(&o, sizeof(float) * 128);
    cudaMemcpy(d, h.data(), sizeof(float) * R * C, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    for (int bh : {1, 4}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
        cuuint64_t strides[1] = {(cuuint64_t)C * 4};
        cuuint32_t box[2] = {32, (cuuint32_t)bh};
        cuuint32_t es[2] = {1, 1};
        CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("box height %d: encode rc=%d\n", bh, (int)rc);
        if (rc) continue;
        cudaMemset(o, 0, sizeof(float) * 128);
        k_probe<<<1, 128>>>(tm, 32, 5, 9, 2, 63, o);
        cudaError_t e = cudaDeviceSynchronize();
        printf("  launch: %s\n", cudaGetErrorString(e));
        if (e) return 1;
        float ho[128];
        cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
        for (int j = 0; j < 4; j++) {
            printf("  row slot %d:", j);
            for (int c = 0; c < 32; c += 4) printf(" %.0f", ho[j * 32 + c]);
            printf("\n");
        }
    }
    return 0;
}
