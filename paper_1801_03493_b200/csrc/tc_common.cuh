// tc_common.cuh -- shared tcgen05 / cp.async / mbarrier helpers of the
// tensor-core kernels (K2a screen_tc.cu, K1b fc_head.cu).
#pragma once

#include <cstdint>

namespace fx {

constexpr int TC_KT = 32;  // K elements (fp32 / tf32) per pipeline stage

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
    // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0) in bits 61..63
    return d;
}

// K-major SWIZZLE_128B operand (TMA tiled boxes of 32 fp32 x rows): SBO =
// 1024 B between 8-row atoms, LBO unused (1), version 1, layout 2.  The K
// slice kk of an atom starts kk * 32 B further.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity));
}

// As mbar_wait, backing off between polls (waiters that would otherwise
// compete for issue slots with the threads they wait for).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    for (;;) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(64);
    }
}

// Operand tile: NR rows x TC_KT floats at k0; row r of the tile -> global row
// pointer rows[r] (nullptr -> zeros).  Canonical no-swizzle K-major layout:
// ((r/8)*(KT/4) + c)*128 + (r%8)*16 (8-row x 16-byte core matrices).
template <int NR, int NT>
__device__ __forceinline__ void load_tile(uint32_t sbase, const float *const *rows, int k0, int D,
                                          const void *dummy) {
    // NR rows x (KT/4 = 8) chunks of 16 bytes over NT threads.  A warp takes
    // 8 rows x 4 chunks: its 32 shared-memory writes fall in 8 distinct
    // 16-byte bank groups (4 wavefronts, the minimum for 512 bytes); 4 rows x
    // 8 chunks would hit only 4 groups (8 wavefronts).
#pragma unroll
    for (int e = 0; e < (NR * TC_KT / 4) / NT; e++) {
        const int idx = threadIdx.x + e * NT;
        const int lane = idx & 31, wq = idx >> 5;
        const int r = ((wq >> 1) << 3) + (lane & 7), c = ((wq & 1) << 2) + (lane >> 3);
        const float *row = rows[r];
        const int k = k0 + c * 4;
        const bool ok = row != nullptr && k < D;
        const void *src = ok ? (const void *)(row + k) : dummy;  // never read when src-size is 0
        const uint32_t dst = sbase + (uint32_t)((((r >> 3) * (TC_KT / 4) + c) << 7) + ((r & 7) << 4));
        cp_async16(dst, src, ok ? 16 : 0);
    }
}


// tcgen05.mma instruction descriptor: D = F32, A = B = TF32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace fx
