// fc_head.cu -- K1b: the cheap-CNN classifier head of the north star
// (no reference function -- it plugs in through the
// reference's classify_fn hook, ingest.py:52-61,73):
//     logits = f W^T + b,  top-K classes by descending logit (ties -> smaller
//     class id), softmax confidences of the K emitted classes.
//
// Two kernels per batch of objects:
//   k_fc_tc    tcgen05.mma kind::tf32, 128 objects x 256 classes per CTA,
//              accumulator in TMEM; the epilogue keeps, per object and class
//              tile, the FC_KC largest TF32 logits, the largest upper bound
//              of every class it dropped (tail), and a logsumexp partial.
//   k_fc_merge one warp per object: candidates whose upper bound reaches the
//              K-th largest lower bound are re-scored in float64 (products
//              of fp32 values are exact in float64; sums round at 2^-53), the
//              top K taken in float64 order.  If a dropped class could still
//              reach the top K (tail >= K-th lower bound) every class is
//              re-scored.  Objects whose float64 logits among ranks 1..K+1
//              are closer than the float64 error bound are flagged (the
//              margin the north star allows; the order of an exact tie is
//              decided by class id as in a stable sort).
// TF32 error bound per logit: |l~ - l| <= gamma ||f|| ||w_v|| + 2^-22 |l~|,
// gamma = 2^-9 + D 2^-22 (as for the distance screen, screen_tc.cu).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "fx_handles.cuh"
#include "tc_common.cuh"

namespace fx {

constexpr int FC_M = 128, FC_N = 256, FC_STAGES = 4, FC_THREADS = 256, FC_KC = 16;
constexpr int FC_A_BYTES = FC_M * TC_KT * 4, FC_B_BYTES = FC_N * TC_KT * 4;

struct FcTile {  // per (object, class tile) result of k_fc_tc
    float val[FC_KC];
    int idx[FC_KC];
    float tail;        // max over dropped classes of (logit~ + err)
    float lse_m, lse_s;  // logsumexp partial: max logit~, sum exp(l~ - max)
};

// TMA = true (objects' rows consecutive in memory): one SWIZZLE_128B tiled
// box per operand and stage (A: 128 rows of tmA from row arow0 + ta, B: 256
// class rows of tmW), issued by one producer thread; one MMA thread; per-
// stage full barriers count bytes, empty barriers take the MMA commit.
// Packed (logit, class) keys of the epilogue; see fc_epilogue.
constexpr float FC_REL = 6.2e-5f;  // relative error of a kept logit: key truncation 2^-15 (x2) + fp32 2^-22
__device__ __forceinline__ int fc_key(float x, int c) {  // c: class within the 256-class tile
    const int b = __float_as_int(x);
    const int o = b < 0 ? b ^ 0x7FFFFFFF : b;  // order-preserving as a signed int
    return (o & ~255) | (255 - c);
}
__device__ __forceinline__ float fc_key_value(int key) {
    const int o = key & ~255;
    return __int_as_float(o < 0 ? o ^ 0x7FFFFFFF : o);
}

// Bitonic sorting network, 16 keys, descending (min/max only).
__device__ __forceinline__ void fc_sort16_desc(int (&a)[16]) {
#pragma unroll
    for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const int l = i ^ j;
                if (l > i) {
                    const int hi = max(a[i], a[l]), lo = min(a[i], a[l]);
                    const bool desc = (i & k) == 0 || k == 16;
                    a[i] = desc ? hi : lo;
                    a[l] = desc ? lo : hi;
                }
            }
}
// kv (16 keys, descending) <- the 16 largest of kv and c (descending); the
// largest key that falls out goes to dropped.
__device__ __forceinline__ void fc_merge16(int (&kv)[16], const int (&c)[16], int &dropped) {
    int m[16];
#pragma unroll
    for (int i = 0; i < 16; i++) {  // kv descending, c reversed ascending: m is bitonic
        m[i] = max(kv[i], c[15 - i]);
        dropped = max(dropped, min(kv[i], c[15 - i]));
    }
#pragma unroll
    for (int j = 8; j > 0; j >>= 1)  // bitonic clean, descending
#pragma unroll
        for (int i = 0; i < 16; i++)
            if ((i & j) == 0) {
                const int hi = max(m[i], m[i + j]), lo = min(m[i], m[i + j]);
                m[i] = hi;
                m[i + j] = lo;
            }
#pragma unroll
    for (int i = 0; i < 16; i++) kv[i] = m[i];
}

// Epilogue of one 128 x 256 accumulator (TMEM columns tmem..tmem+255): 256
// threads, warps (quad, half): TMEM lanes 32 quad.. (object rows) and one half
// of the 256 classes each; a thread keeps the FC_KC largest logits of its
// half (sorted descending, ties -> smaller class id), the largest dropped
// logit and a logsumexp partial, then the upper half hands its list to the
// lower one through shared memory (its class ids are all larger, so
// inserting after keeps the tie order).  The tail (largest upper bound of a
// dropped class) uses the tile's largest ||w||.  out: this class tile's
// FcTile of object 0 (stride ntile per object).  tmem_empty: arrived on by
// every thread once the accumulator is read (persistent kernel).
template <class Sync>
__device__ __forceinline__ void fc_epilogue(uint32_t tmem, int quad, int half, int lane, int etid, int ta, int tv,
                                            int n, int64_t a0, int V, const float *__restrict__ fnorm,
                                            const float *__restrict__ wnorm, const float *__restrict__ bias,
                                            float gamma, FcTile *__restrict__ out, int ntile, float *s_wmax, float *s_bias,
                                            float *hv, int *hi, float *hx, uint64_t *tmem_empty, Sync sync,
                                            int edbg = 0) {
    const int a = ta + quad * 32 + lane;
    const float fn = a < n ? fnorm[a0 + a] : 0.f;
    {
        float wm = tv + etid < V ? wnorm[tv + etid] : 0.f;  // 256 epilogue threads, 256 classes
        s_bias[etid] = bias && tv + etid < V ? bias[tv + etid] : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        if (lane == 0) s_wmax[etid >> 5] = wm;
        sync();
    }
    float wmax = 0.f;
#pragma unroll
    for (int w = 0; w < 8; w++) wmax = fmaxf(wmax, s_wmax[w]);
    // Kept logits as packed keys: the float's order-preserving int with the
    // low 8 bits replaced by 255 - (class within the tile), so one signed
    // compare orders by value and then by smaller class id; the dropped bits
    // cost < 2^-15 |logit| (FC_REL covers it).  Keys are unique within the
    // tile, so the kept set and the largest dropped key do not depend on the
    // order of insertion: 16 keys at a time are sorted by a bitonic network
    // and merged into the list (fc_merge16) -- min/max only, no divergence
    // between the lanes (objects) of a warp.
    int kv[FC_KC];
#pragma unroll
    for (int j = 0; j < FC_KC; j++) kv[j] = INT_MIN;
    int dropped = INT_MIN;
    auto tmem_row = [&](int c0, uint32_t *v) {
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
    };
    constexpr int HC = FC_N / 2;
    float m = -FLT_MAX, ssum = 0.f;  // logsumexp partial, updated per 32-class chunk (one TMEM pass)
    for (int c0 = half * HC; c0 < (half + 1) * HC; c0 += 32) {
        uint32_t v[32];
        tmem_row(c0, v);
        float x[32];
        float cm = -FLT_MAX;
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const int cls = tv + c0 + j;
            x[j] = (a < n && cls < V) ? __uint_as_float(v[j]) + s_bias[c0 + j] : -FLT_MAX;
            cm = fmaxf(cm, x[j]);
        }
        if (cm != -FLT_MAX) {  // else past the last class (or object); no divergent exit before tcgen05.ld
            const float nm = fmaxf(m, cm);
            float cs = 0.f;
#pragma unroll
            for (int j = 0; j < 32; j++) cs += (edbg & 32) || x[j] == -FLT_MAX ? 0.f : __expf(x[j] - nm);
            ssum = ssum * __expf(m - nm) + cs;
            m = nm;
            if (!(edbg & 16)) {
#pragma unroll
                for (int h = 0; h < 32; h += 16) {  // 16 keys at a time: sort them, merge into the list
                    int c[16];
#pragma unroll
                    for (int i = 0; i < 16; i++) c[i] = x[h + i] != -FLT_MAX ? fc_key(x[h + i], c0 + h + i) : INT_MIN;
                    fc_sort16_desc(c);
                    fc_merge16(kv, c, dropped);
                }
            }
        }
    }
    if (tmem_empty) {  // accumulator read: the MMA may overwrite it
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_empty)) : "memory");
    }
    // upper half -> lower half through shared memory
    const int r = quad * 32 + lane;
    int *hk = (int *)hv;
    sync();
    if (half == 1) {
#pragma unroll
        for (int j = 0; j < FC_KC; j++) hk[r * FC_KC + j] = kv[j];
        hx[r * 3 + 0] = __int_as_float(dropped);
        hx[r * 3 + 1] = m;
        hx[r * 3 + 2] = ssum;
    }
    sync();
    if (half == 0) {
        int c[FC_KC];
#pragma unroll
        for (int j = 0; j < FC_KC; j++) c[j] = hk[r * FC_KC + j];  // sorted (descending) already
        fc_merge16(kv, c, dropped);
        dropped = max(dropped, __float_as_int(hx[r * 3 + 0]));
        const float m1 = hx[r * 3 + 1], s1 = hx[r * 3 + 2];
        const float mm = fmaxf(m, m1);
        ssum = (ssum > 0.f ? ssum * __expf(m - mm) : 0.f) + (s1 > 0.f ? s1 * __expf(m1 - mm) : 0.f);
        const float dv = fc_key_value(dropped);
        const float tail = dropped == INT_MIN ? -FLT_MAX : dv + gamma * fn * wmax + fabsf(dv) * FC_REL;
        if (a < n) {
            FcTile *o = out + (int64_t)a * ntile;
#pragma unroll
            for (int j = 0; j < FC_KC; j++) {
                o->val[j] = kv[j] == INT_MIN ? -FLT_MAX : fc_key_value(kv[j]);
                o->idx[j] = kv[j] == INT_MIN ? -1 : tv + 255 - (kv[j] & 255);
            }
            o->tail = tail;
            o->lse_m = mm;
            o->lse_s = ssum;
        }
    }
    sync();  // hv / s_wmax free for the next tile
}

//
// CL > 1 (TMA only): the CTAs of a (1, CL) cluster share one class tile and
// take CL consecutive object tiles; each loads 256/CL rows of the W box and
// multicasts them to every CTA of the cluster, so a CTA pulls 1 + 2/CL MB
// from L2 per (128 objects x 256 classes x 2048) tile instead of 3 MB.  A
// stage is free again when all CL MMAs consumed it (each MMA commit arrives
// on every CTA's empty barrier, count CL).
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <bool TMA, int CL>
__global__ void __launch_bounds__(FC_THREADS, 1) k_fc_tc(int n, int64_t a0, const char *const *__restrict__ frow,
                                                        const float *__restrict__ fnorm, int D, int V,
                                                        const float *__restrict__ W, const float *__restrict__ wnorm,
                                                        const float *__restrict__ bias, float gamma,
                                                        FcTile *__restrict__ out, int dbg,
                                                        const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmW, int arow0) {
    const int tv = blockIdx.x * FC_N, ta = blockIdx.y * FC_M;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // SWIZZLE_128B atoms
    __shared__ const float *rowsA[FC_M];
    __shared__ const float *rowsB[FC_N];
    __shared__ __align__(8) uint64_t bar_stage[FC_STAGES];
    __shared__ __align__(8) uint64_t bar_full[FC_STAGES];
    __shared__ __align__(8) uint64_t bar_done;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (!TMA) {
        for (int r = tid; r < FC_M; r += FC_THREADS) rowsA[r] = ta + r < n ? (const float *)frow[a0 + ta + r] : nullptr;
        for (int r = tid; r < FC_N; r += FC_THREADS) rowsB[r] = tv + r < V ? W + (int64_t)(tv + r) * D : nullptr;
    }
    if (tid == 0) {
        for (int s = 0; s < FC_STAGES; s++) {
            mbar_init(&bar_stage[s], CL);
            mbar_init(&bar_full[s], 1);
        }
        mbar_init(&bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    uint32_t crank = 0;
    if (CL > 1) {
        asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
        cluster_sync_all();  // peers' barriers initialised before any multicast lands
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "r"(FC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    const uint32_t tmem = tmem_base;
    const uint32_t sbase = smem_u32(smem);
    const int nk = (D + TC_KT - 1) / TC_KT;
    constexpr uint32_t idesc = idesc_tf32(FC_M, FC_N);
    constexpr int SB = FC_A_BYTES + FC_B_BYTES;
    if (TMA) {
        if (warp == 0 && lane == 0) {  // producer
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmW) : "memory");
            for (int it = 0; it < nk; it++) {
                const int s = it % FC_STAGES;
                if (it >= FC_STAGES) mbar_wait(&bar_stage[s], (uint32_t)(((it / FC_STAGES) - 1) & 1));
                const uint32_t st = sbase + s * SB, fb = smem_u32(&bar_full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(SB) : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3}], [%4];\n" ::"r"(st),
                    "l"(&tmA), "r"(it * TC_KT), "r"(arow0 + ta), "r"(fb)
                    : "memory");
                if (CL == 1) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
                        "{%2, %3}], [%4];\n" ::"r"(st + FC_A_BYTES),
                        "l"(&tmW), "r"(it * TC_KT), "r"(tv), "r"(fb)
                        : "memory");
                } else {
                    constexpr int WR = FC_N / CL;  // W rows this CTA fetches for the whole cluster
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::"
                        "cluster [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(st + FC_A_BYTES + crank * (WR * TC_KT * 4)),
                        "l"(&tmW), "r"(it * TC_KT), "r"(tv + (int)crank * WR), "r"(fb), "h"((uint16_t)((1u << CL) - 1u))
                        : "memory");
                }
            }
        } else if (warp == 1 && lane == 0) {  // MMA issue
            for (int it = 0; it < nk; it++) {
                const int s = it % FC_STAGES;
                mbar_wait(&bar_full[s], (uint32_t)((it / FC_STAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
                const uint32_t st = sbase + s * SB;
#pragma unroll
                for (int kk = 0; kk < TC_KT / 8; kk++) {
                    const uint64_t da = umma_desc_sw128(st + kk * 32);
                    const uint64_t db = umma_desc_sw128(st + FC_A_BYTES + kk * 32);
                    const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                        "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
                if (CL == 1)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&bar_stage[s])));
                else
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                        "%1;\n" ::"r"(smem_u32(&bar_stage[s])),
                        "h"((uint16_t)((1u << CL) - 1u)));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&bar_done)));
        }
    } else {
        for (int s = 0; s < FC_STAGES - 1; s++) {
            if (s < nk && !(dbg & 1)) {
                load_tile<FC_M, FC_THREADS>(sbase + s * SB, rowsA, s * TC_KT, D, fnorm);
                load_tile<FC_N, FC_THREADS>(sbase + s * SB + FC_A_BYTES, rowsB, s * TC_KT, D, fnorm);
            }
            asm volatile("cp.async.commit_group;\n" ::);
        }
        for (int it = 0; it < nk; it++) {
            const int s = it % FC_STAGES;
            asm volatile("cp.async.wait_group %0;\n" ::"n"(FC_STAGES - 2));
            asm volatile("fence.proxy.async.shared::cta;\n" ::);
            __syncthreads();
            if (tid == 0 && !(dbg & 2)) {
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
                const uint32_t st = sbase + s * SB;
#pragma unroll
                for (int kk = 0; kk < TC_KT / 8; kk++) {
                    const uint64_t da = umma_desc(st + kk * 256, 128, TC_KT * 32);
                    const uint64_t db = umma_desc(st + FC_A_BYTES + kk * 256, 128, TC_KT * 32);
                    const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                        "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&bar_stage[s])));
            }
            const int nt = it + FC_STAGES - 1;
            if (nt < nk) {
                const int ns = nt % FC_STAGES;
                if (nt >= FC_STAGES && !(dbg & 2)) mbar_wait(&bar_stage[ns], (uint32_t)(((nt / FC_STAGES) - 1) & 1));
                if (!(dbg & 1)) {
                    load_tile<FC_M, FC_THREADS>(sbase + ns * SB, rowsA, nt * TC_KT, D, fnorm);
                    load_tile<FC_N, FC_THREADS>(sbase + ns * SB + FC_A_BYTES, rowsB, nt * TC_KT, D, fnorm);
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        }
        if (tid == 0 && !(dbg & 2))
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&bar_done)));
    }
    if (!(dbg & 2)) mbar_wait(&bar_done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);

    // epilogue: warps w and w+4 share TMEM lanes 32(w%4).. (object rows) and
    // take one half of the 256 classes each; a thread keeps the FC_KC largest
    // logits of its half (sorted descending, ties -> smaller class id), the
    // largest dropped logit and a logsumexp partial, then the upper half hands
    // its list to the lower one through shared memory (its class ids are all
    // larger, so inserting after keeps the tie order).  The tail (largest
    // upper bound of a dropped class) uses the tile's largest ||w||.
    if (!(dbg & 4)) {  // dbg & 4: main loop only (timing experiments)
        __shared__ float s_wmax[8], s_bias[FC_N];
        float *hv = (float *)smem;  // the pipeline's shared memory is idle now
        fc_epilogue(tmem, warp & 3, warp >> 2, lane, tid, ta, tv, n, a0, V, fnorm, wnorm, bias, gamma,
                    out + blockIdx.x, gridDim.x, s_wmax, s_bias, hv, (int *)(hv + FC_M * FC_KC),
                    (float *)(hv + 2 * FC_M * FC_KC), nullptr, [] { __syncthreads(); });
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
    if (CL > 1) cluster_sync_all();  // no peer still multicasts into this CTA's stages or barriers
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(FC_N));
}

// Persistent K1b logits (TMA operands): one CTA per SM walks the (object
// tile, class tile) pairs t = blockIdx.x + i gridDim.x, class tile fastest
// (CTAs running at the same time share object rows in L2).  Warp 0 lane 0
// streams the operands through the FC_STAGES ring, warp 1 lane 0 issues the
// MMAs into one of two TMEM accumulators (2 x 256 columns), warps 4..11 run
// fc_epilogue on the other: tile i's epilogue overlaps tile i+1's main loop.
// Barriers: full/empty per stage (as k_fc_tc), acc_full[b] (MMA commit ->
// epilogue), acc_empty[b] (256 epilogue arrivals -> MMA).
constexpr int FCP_THREADS = 384;
__global__ void __launch_bounds__(FCP_THREADS, 1) k_fc_tcp(int n, int64_t a0, const float *__restrict__ fnorm, int D,
                                                          int V, const float *__restrict__ wnorm,
                                                          const float *__restrict__ bias, float gamma,
                                                          FcTile *__restrict__ out, int ntile, int ntiles,
                                                          const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmW, int arow0,
                                                          int dbg) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar_empty[FC_STAGES];
    __shared__ __align__(8) uint64_t bar_full[FC_STAGES];
    __shared__ __align__(8) uint64_t acc_full[2];
    __shared__ __align__(8) uint64_t acc_empty[2];
    __shared__ float s_wmax[8], s_bias[FC_N];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int SB = FC_A_BYTES + FC_B_BYTES;
    float *hv = (float *)(smem + FC_STAGES * SB);  // [128][FC_KC] vals, [128][FC_KC] ids, [128][3]
    if (tid == 0) {
        for (int s = 0; s < FC_STAGES; s++) {
            mbar_init(&bar_empty[s], 1);
            mbar_init(&bar_full[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "r"(2 * FC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    const uint32_t tmem = tmem_base;
    const uint32_t sbase = smem_u32(smem);
    const int nk = (D + TC_KT - 1) / TC_KT;
    constexpr uint32_t idesc = idesc_tf32(FC_M, FC_N);
    if (warp == 0 && lane == 0) {  // producer
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmW) : "memory");
        uint32_t g = 0;  // stage uses so far
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int tv = (t % ntile) * FC_N, ta = (t / ntile) * FC_M;
            for (int it = 0; it < nk; it++, g++) {
                const int s = g % FC_STAGES;
                mbar_wait(&bar_empty[s], ((g / FC_STAGES) + 1) & 1);
                const uint32_t st = sbase + s * SB, fb = smem_u32(&bar_full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(SB) : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3}], [%4];\n" ::"r"(st),
                    "l"(&tmA), "r"(it * TC_KT), "r"(arow0 + ta), "r"(fb)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3}], [%4];\n" ::"r"(st + FC_A_BYTES),
                    "l"(&tmW), "r"(it * TC_KT), "r"(tv), "r"(fb)
                    : "memory");
            }
        }
    } else if (warp == 1 && lane == 0) {  // MMA issue
        uint32_t g = 0, i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, i++) {
            const uint32_t b = i & 1, acc_t = tmem + b * FC_N;
            mbar_wait(&acc_empty[b], ((i >> 1) + 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
            for (int it = 0; it < nk; it++, g++) {
                const int s = g % FC_STAGES;
                mbar_wait(&bar_full[s], (g / FC_STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
                const uint32_t st = sbase + s * SB;
#pragma unroll
                for (int kk = 0; kk < TC_KT / 8; kk++) {
                    const uint64_t da = umma_desc_sw128(st + kk * 32);
                    const uint64_t db = umma_desc_sw128(st + FC_A_BYTES + kk * 32);
                    const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc_t),
                        "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&bar_empty[s])));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&acc_full[b])));
        }
    } else if (warp >= 4) {  // epilogue
        const int ew = warp - 4, etid = tid - 128;
        uint32_t i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, i++) {
            const int ct = t % ntile, tv = ct * FC_N, ta = (t / ntile) * FC_M;
            const uint32_t b = i & 1;
            if (lane == 0) mbar_wait_sleep(&acc_full[b], (i >> 1) & 1);  // one waiter per warp
            __syncwarp();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
            if (dbg & 4) {  // main loop only (timing experiments)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&acc_empty[b])) : "memory");
                continue;
            }
            fc_epilogue(tmem + b * FC_N, ew & 3, ew >> 2, lane, etid, ta, tv, n, a0, V, fnorm, wnorm, bias, gamma,
                        out + ct, ntile, s_wmax, s_bias, hv, (int *)(hv + FC_M * FC_KC), (float *)(hv + 2 * FC_M * FC_KC),
                        &acc_empty[b], [] { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }, dbg);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * FC_N));
}

// float64 logit of class v for feature row f (warp-cooperative; result in all lanes)
// (rows 16-byte aligned, D % 4 == 0: float4 loads, two independent chains per lane)
template <int FC_LD>  // 16-byte chunks of each row per lane in flight
__device__ __forceinline__ double fc_logit64(const float *f, const float *w, int D, double b) {
    const float4 *f4 = (const float4 *)f, *w4 = (const float4 *)w;
    double acc[8];
#pragma unroll
    for (int e = 0; e < 8; e++) acc[e] = 0.0;
    const int n4 = D >> 2;
    int k = threadIdx.x & 31;
    for (; k + 32 * (FC_LD - 1) < n4; k += 32 * FC_LD) {  // FC_LD 16-byte chunks of each row per lane in flight
        float4 x[FC_LD], y[FC_LD];
#pragma unroll
        for (int u = 0; u < FC_LD; u++) {
            y[u] = __ldg(w4 + k + 32 * u);
            x[u] = __ldg(f4 + k + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < FC_LD; u++) {
            double *a = acc + 4 * (u & 1);
            a[0] = fma((double)x[u].x, (double)y[u].x, a[0]);
            a[1] = fma((double)x[u].y, (double)y[u].y, a[1]);
            a[2] = fma((double)x[u].z, (double)y[u].z, a[2]);
            a[3] = fma((double)x[u].w, (double)y[u].w, a[3]);
        }
    }
    for (; k < n4; k += 32) {
        const float4 x = __ldg(f4 + k), y = __ldg(w4 + k);
        acc[0] = fma((double)x.x, (double)y.x, acc[0]);
        acc[1] = fma((double)x.y, (double)y.y, acc[1]);
        acc[2] = fma((double)x.z, (double)y.z, acc[2]);
        acc[3] = fma((double)x.w, (double)y.w, acc[3]);
    }
    double r = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r + b;
}

// The float64 logit as fc_logit64 (eight partial sums per lane), the feature row held in registers (fr[i] = f4[lane
// + 32 i], i < nf = D / 128 <= 16): per candidate only the W row is loaded,
// 8 float4 per lane in flight.
template <bool REG>
__device__ __forceinline__ double fc_logit64_reg(const float4 (&fr)[REG ? 16 : 1], int nf, const float *w, double b) {
    const float4 *w4 = (const float4 *)w;
    const int lane = threadIdx.x & 31;
    double acc[8];  // eight independent FMA chains (a chain of 64 dependent DFMAs stalls the warp)
#pragma unroll
    for (int e = 0; e < 8; e++) acc[e] = 0.0;
#pragma unroll
    for (int h = 0; h < 16; h += 8) {
        if (h >= nf) break;
        float4 y[8];
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (h + i < nf) y[i] = __ldg(w4 + lane + 32 * (h + i));
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (h + i < nf) {
                const float4 x = fr[REG ? h + i : 0];
                double *a = acc + 4 * (i & 1);
                a[0] = fma((double)x.x, (double)y[i].x, a[0]);
                a[1] = fma((double)x.y, (double)y[i].y, a[1]);
                a[2] = fma((double)x.z, (double)y[i].z, a[2]);
                a[3] = fma((double)x.w, (double)y[i].w, a[3]);
            }
    }
    double r = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r + b;
}

constexpr int FC_MAXC = 64;  // candidates re-scored per object before the all-class fallback
#ifndef FC_MERGE_MINB
#define FC_MERGE_MINB 4  // merge CTAs per SM (registers <= 64: the re-score is latency-bound)
#endif

template <bool REG, int LD>
__global__ void __launch_bounds__(256, REG ? 2 : FC_MERGE_MINB) k_fc_merge(int n, int64_t a0, const char *const *__restrict__ frow,
                                                 const int64_t *__restrict__ cls_obj, const float *__restrict__ fnorm,
                                                 int D, int V, int K, const float *__restrict__ W,
                                                 const float *__restrict__ wnorm, const float *__restrict__ bias,
                                                 float gamma, int ntile, const FcTile *__restrict__ tiles,
                                                 int32_t *__restrict__ topk, float *__restrict__ conf,
                                                 uint8_t *__restrict__ flag, unsigned long long *__restrict__ nflag,
                                                 unsigned long long *stats) {
    __shared__ int s_idx[8][FC_MAXC];
    __shared__ float s_lb[8][FC_MAXC], s_ub[8][FC_MAXC];
    __shared__ unsigned char s_need[8][FC_MAXC];
    __shared__ double s_bv[8][17];
    __shared__ int s_bi[8][17];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w = blockIdx.x * 8 + wib;
    if (w >= n) return;
    const float fn = fnorm[a0 + w];
    const float *f = (const float *)frow[a0 + w];
    const FcTile *t = tiles + (int64_t)w * ntile;
    // K-th largest lower bound among the tiles' kept candidates (K rounds of
    // warp argmax), then the candidates: kept classes whose upper bound reaches
    // it.  With <= 64 kept entries (V <= 1024) each lane holds its two in
    // registers; otherwise the entries are re-read per round.
    const int nc = ntile * FC_KC;
    float lbk = -FLT_MAX;
    float maxtail = -FLT_MAX;
    for (int ti = 0; ti < ntile; ti++) maxtail = fmaxf(maxtail, t[ti].tail);
    bool all;
    int ncand = 0;
    if (nc <= 64) {
        int ecls[2];
        float elv[2], elb[2], eub[2], ekb[2];  // ekb: the ranking bound, rounded as in the general path
        bool taken[2] = {false, false};
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int e = lane + 32 * u;
            ecls[u] = e < nc ? t[e / FC_KC].idx[e % FC_KC] : -1;
            elv[u] = e < nc ? t[e / FC_KC].val[e % FC_KC] : 0.f;
            const float ge = ecls[u] >= 0 ? gamma * fn * wnorm[ecls[u]] : 0.f;
            const float err = ge + fabsf(elv[u]) * FC_REL;
            ekb[u] = elv[u] - ge - fabsf(elv[u]) * FC_REL;
            elb[u] = elv[u] - err;
            eub[u] = elv[u] + err;
        }
        for (int r = 0; r < K; r++) {
            float best = -FLT_MAX;
            int bslot = -1;
#pragma unroll
            for (int u = 0; u < 2; u++)
                if (ecls[u] >= 0 && !taken[u] && ekb[u] > best) {
                    best = ekb[u];
                    bslot = lane + 32 * u;
                }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int os = __shfl_xor_sync(0xffffffffu, bslot, o);
                if (ob > best || (ob == best && os >= 0 && (bslot < 0 || os < bslot))) {
                    best = ob;
                    bslot = os;
                }
            }
            if (bslot == lane) taken[0] = true;
            if (bslot == lane + 32) taken[1] = true;
            lbk = best;
        }
        all = maxtail >= lbk;
        if (!all) {
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const bool take = ecls[u] >= 0 && eub[u] >= lbk;
                const unsigned m = __ballot_sync(0xffffffffu, take);
                if (take) {
                    const int pos = ncand + __popc(m & ((1u << lane) - 1u));
                    if (pos < FC_MAXC) {
                        s_idx[wib][pos] = ecls[u];
                        s_lb[wib][pos] = elb[u];
                        s_ub[wib][pos] = eub[u];
                    }
                }
                ncand += __popc(m);
            }
            if (ncand > FC_MAXC) all = true;
        }
    } else {
        for (int r = 0; r < K; r++) {
            float best = -FLT_MAX;
            int bslot = -1;
            for (int e = lane; e < nc; e += 32) {
                const int ti = e / FC_KC, j = e % FC_KC;
                const int cls = t[ti].idx[j];
                if (cls < 0) continue;
                bool done = false;
                for (int q = 0; q < r; q++) done |= (s_idx[wib][q] == e);
                const float lv = t[ti].val[j];
                const float lb = lv - gamma * fn * wnorm[cls] - fabsf(lv) * FC_REL;
                if (!done && lb > best) {
                    best = lb;
                    bslot = e;
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int os = __shfl_xor_sync(0xffffffffu, bslot, o);
                if (ob > best || (ob == best && os >= 0 && (bslot < 0 || os < bslot))) {
                    best = ob;
                    bslot = os;
                }
            }
            __syncwarp();
            if (lane == 0) s_idx[wib][r] = bslot;
            __syncwarp();
            lbk = best;
        }
        all = maxtail >= lbk;
        if (!all) {
            for (int e0 = 0; e0 < nc; e0 += 32) {
                const int e = e0 + lane;
                bool take = false;
                int cls = -1;
                if (e < nc) {
                    const int ti = e / FC_KC, j = e % FC_KC;
                    cls = t[ti].idx[j];
                    if (cls >= 0) {
                        const float lv = t[ti].val[j];
                        take = lv + gamma * fn * wnorm[cls] + fabsf(lv) * FC_REL >= lbk;
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, take);
                if (take) {
                    const int pos = ncand + __popc(m & ((1u << lane) - 1u));
                    if (pos < FC_MAXC) {
                        const int ti = e / FC_KC, j = e % FC_KC;
                        const float lv = t[ti].val[j];
                        const float err = gamma * fn * wnorm[cls] + fabsf(lv) * FC_REL;
                        s_idx[wib][pos] = cls;
                        s_lb[wib][pos] = lv - err;
                        s_ub[wib][pos] = lv + err;
                    }
                }
                ncand += __popc(m);
            }
            if (ncand > FC_MAXC) all = true;
        }
    }
    __syncwarp();
    // only candidates whose TF32 interval overlaps another candidate's need
    // their float64 value: disjoint intervals are already ordered (and far
    // outside the float64 margin)
    if (!all) {
        for (int c = lane; c < ncand; c += 32) {
            bool ov = false;
            for (int o = 0; o < ncand; o++)
                ov |= o != c && s_lb[wib][o] <= s_ub[wib][c] && s_lb[wib][c] <= s_ub[wib][o];
            s_need[wib][c] = ov ? 1 : 0;
        }
        __syncwarp();
    }
    // float64 re-score, selection of the top K (+1 for the margin check):
    // the sorted list lives in shared memory, lane 0 inserts
    double *bv = s_bv[wib];
    int *bi = s_bi[wib];
    const int K1 = K + 1 < 17 ? K + 1 : 17;
    if (lane < 17) {
        bv[lane] = -DBL_MAX;
        bi[lane] = INT_MAX;
    }
    __syncwarp();
    const int nscore = all ? V : ncand;
    const bool reg = REG && (D & 127) == 0 && D <= 2048;  // feature row cached in registers
    const int nf = D >> 7;
    float4 fr[REG ? 16 : 1];
    if (REG && reg) {
#pragma unroll
        for (int i = 0; i < 16; i++)
            if (i < nf) fr[i] = __ldg((const float4 *)f + lane + 32 * i);
    }
    for (int c = 0; c < nscore; c++) {
        const int cls = all ? c : s_idx[wib][c];
        double l;
        if (all || s_need[wib][c])
            l = reg ? fc_logit64_reg<REG>(fr, nf, W + (int64_t)cls * D, bias ? (double)bias[cls] : 0.0)
                    : fc_logit64<LD>(f, W + (int64_t)cls * D, D, bias ? (double)bias[cls] : 0.0);
        else
            l = 0.5 * ((double)s_lb[wib][c] + (double)s_ub[wib][c]);  // disjoint interval: its order is certain
        if (lane == 0) {  // lane 0's value decides (its reduction order is fixed)
            double x = l;
            int xi = cls;
            for (int q = 0; q < K1; q++) {
                if (x > bv[q] || (x == bv[q] && xi < bi[q])) {
                    const double tv = bv[q];
                    const int ti = bi[q];
                    bv[q] = x;
                    bi[q] = xi;
                    x = tv;
                    xi = ti;
                }
            }
        }
        __syncwarp();
    }
    // margin flag: the float64 error of a logit is <= (D + 8) 2^-53 ||f|| ||w|| + the bias add
    bool flagged = false;
    const double ue = ((double)D + 8.0) * 1.1102230246251565e-16 * (double)fn * 1.0001;
    if (lane == 0)
        for (int q = 0; q + 1 < K1 && q + 1 < nscore; q++) {
            const double e1 = ue * (double)wnorm[bi[q]] + fabs(bv[q]) * 2.3e-16;
            const double e2 = ue * (double)wnorm[bi[q + 1]] + fabs(bv[q + 1]) * 2.3e-16;
            if (bv[q] - bv[q + 1] <= 2.0 * (e1 + e2)) flagged = true;
        }
    if (lane == 0) {
        // logsumexp over all classes from the tiles' partials (TF32 logits; confidences only)
        float M = -FLT_MAX;
        for (int ti = 0; ti < ntile; ti++) M = fmaxf(M, t[ti].lse_m);
        float S = 0.f;
        for (int ti = 0; ti < ntile; ti++) S += t[ti].lse_s * __expf(t[ti].lse_m - M);
        const float lse = M + __logf(S);
        const int64_t obj = cls_obj ? cls_obj[a0 + w] : a0 + w;
        for (int j = 0; j < K; j++) {
            topk[obj * K + j] = bi[j];
            if (conf) conf[obj * K + j] = __expf((float)bv[j] - lse);
        }
        if (flag) flag[obj] = flagged ? 1 : 0;
        if (flagged && nflag) atomicAdd(nflag, 1ull);
        if (stats) {  // FOCUS_B200_FC_STATS: objects re-scored over every class / candidates re-scored
            atomicAdd(stats, all ? 1ull : 0ull);
            unsigned long long nr = 0;
            for (int c = 0; c < ncand && !all; c++) nr += s_need[wib][c];
            atomicAdd(stats + 1, all ? (unsigned long long)V : nr);
            atomicAdd(stats + 2, all ? 0ull : (unsigned long long)(ncand > 64 ? 64 : ncand));
        }
    }
}

__global__ void k_row_norms(int64_t rows, int D, const float *__restrict__ X, float *__restrict__ out) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    float acc = 0.f;
    for (int k = lane; k < D; k += 32) acc = fmaf(X[w * D + k], X[w * D + k], acc);
    acc = warp_sum(acc);
    if (lane == 0) out[w] = sqrtf(acc) * 1.00001f;  // rounded up: an upper bound of ||w||
}

bool make_rows_map(CUtensorMap *tm, const void *base, int64_t rows, int D, int64_t row_bytes, int box_rows);

static int num_sms() {
    static int v[64] = {};
    int &x = v[dev_slot()];
    if (!x) {
        int dev = 0;
        FX_CUDA(cudaGetDevice(&dev));
        FX_CUDA(cudaDeviceGetAttribute(&x, cudaDevAttrMultiProcessorCount, dev));
    }
    return x;
}

// K1b over classified objects [c0, c0 + n) of a stream (topk written by object index).
// Xdense: when the n objects' rows are the consecutive fp32 rows Xdense[0..n)
// (standalone head, compact ingest), operands are staged by TMA.
void launch_fc_head(int64_t n, int64_t c0, const char *const *frow, const int64_t *cls_obj, const float *fnorm, int D,
                    int V, int K, const float *W, const float *wnorm, const float *bias, int32_t *topk, float *conf,
                    uint8_t *flag, unsigned long long *nflag, cudaStream_t st, const float *Xdense) {
    if (n <= 0) return;
    if (K > 16 || K > V) throw Error{FX_E_K_OUT_OF_RANGE, "fc head: k must be <= min(16, vocab)"};
    static bool attr_set[64] = {};
    bool &attr = attr_set[dev_slot()];
    const size_t smem = (size_t)FC_STAGES * (FC_A_BYTES + FC_B_BYTES) + 1024;
    const size_t smem_p = smem + (size_t)FC_M * (2 * FC_KC + 3) * 4;  // + the epilogue's hand-off
    // persistent kernel (TMA operands): FOCUS_B200_FC_PERSIST=0 -> one CTA per tile
    static const bool persist = !(getenv("FOCUS_B200_FC_PERSIST") && atoi(getenv("FOCUS_B200_FC_PERSIST")) == 0);
    if (!attr) {
        for (auto k : {k_fc_tc<false, 1>, k_fc_tc<true, 1>, k_fc_tc<true, 2>, k_fc_tc<true, 4>})
            FX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FX_CUDA(cudaFuncSetAttribute(k_fc_tcp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
        attr = true;
    }
    static const bool tma_off = getenv("FOCUS_B200_TCLOAD") && std::string(getenv("FOCUS_B200_TCLOAD")) == "cp";
    // W multicast cluster size (FOCUS_B200_FC_CL: 1, 2 or 4; default 1: 4 measured
    // 17% slower -- the head is not bound by L2 -> SM operand traffic)
    static const int cl_env = getenv("FOCUS_B200_FC_CL") ? atoi(getenv("FOCUS_B200_FC_CL")) : 1;
    // float64 re-score: the feature row re-read per candidate (L1) at 64 registers, 4 CTAs per SM
    // (FOCUS_B200_FC_MERGE_REG=1: the row held in registers, 2 CTAs per SM -- measured 818 vs 531 us)
    static const int merge_reg = getenv("FOCUS_B200_FC_MERGE_REG") ? atoi(getenv("FOCUS_B200_FC_MERGE_REG")) : 0;
    // row chunks in flight per lane in the re-score (FOCUS_B200_FC_LD: 2 or 4)
    static const int merge_ld = getenv("FOCUS_B200_FC_LD") ? atoi(getenv("FOCUS_B200_FC_LD")) : 4;
    const int CL = (cl_env == 2 || cl_env == 4) ? cl_env : 1;
    CUtensorMap tmA = {}, tmW = {};
    const bool tma = Xdense && !tma_off && D % 4 == 0 && make_rows_map(&tmA, Xdense, n, D, (int64_t)D * 4, FC_M) &&
                     make_rows_map(&tmW, W, V, D, (int64_t)D * 4, FC_N / CL);
    const int ntile = (int)cdiv(V, FC_N);
    const float gamma = (float)((1.953125e-03 + (double)D * 2.384185791015625e-07) * 1.01);
    static const bool fc_stats = getenv("FOCUS_B200_FC_STATS") != nullptr;
    DevBuf<unsigned long long> stats;
    if (fc_stats) {
        stats.reserve(3);
        FX_CUDA(cudaMemsetAsync(stats.p, 0, 3 * sizeof(unsigned long long), st));
    }
    DevBuf<FcTile> tiles;
    const int64_t CH = 1 << 16;  // objects per pass (bounds the tile scratch)
    tiles.reserve((size_t)std::min<int64_t>(n, CH) * ntile);
    for (int64_t b = 0; b < n; b += CH) {
        const int64_t m = std::min<int64_t>(CH, n - b);
        static const int dbg = getenv("FOCUS_B200_FCDBG") ? atoi(getenv("FOCUS_B200_FCDBG")) : 0;
        if (tma && persist && CL == 1) {
            const int ntiles = ntile * (int)cdiv(m, FC_M);
            const int grid = std::min(ntiles, num_sms());
            k_fc_tcp<<<grid, FCP_THREADS, smem_p, st>>>((int)m, c0 + b, fnorm, D, V, wnorm, bias, gamma, tiles.p,
                                                        ntile, ntiles, tmA, tmW, (int)b, dbg);
        } else if (tma && CL > 1) {
            // object tiles padded to whole clusters (TMA zero-fills rows past the
            // features; the padded tiles write nothing)
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)ntile, (unsigned)(cdiv(cdiv(m, FC_M), CL) * CL));
            cfg.blockDim = dim3(FC_THREADS);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1;
            at[0].val.clusterDim.y = (unsigned)CL;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            FX_CUDA(cudaLaunchKernelEx(&cfg, CL == 2 ? k_fc_tc<true, 2> : k_fc_tc<true, 4>, (int)m, c0 + b, frow,
                                       fnorm, D, V, W, wnorm, bias, gamma, tiles.p, dbg, tmA, tmW, (int)b));
        } else {
            dim3 grid((unsigned)ntile, (unsigned)cdiv(m, FC_M));
            (tma ? k_fc_tc<true, 1> : k_fc_tc<false, 1>)<<<grid, FC_THREADS, smem, st>>>(
                (int)m, c0 + b, frow, fnorm, D, V, W, wnorm, bias, gamma, tiles.p, dbg, tmA, tmW, (int)b);
        }
        FX_LAUNCHED();
        (merge_reg ? k_fc_merge<true, 2> : merge_ld == 2 ? k_fc_merge<false, 2> : k_fc_merge<false, 4>)<<<(unsigned)cdiv(m, 8), 256, 0, st>>>((int)m, c0 + b, frow, cls_obj, fnorm, D, V, K, W, wnorm, bias,
                                                        gamma, ntile, tiles.p, topk, conf, flag, nflag,
                                                        fc_stats ? stats.p : nullptr);
        FX_LAUNCHED();
    }
    if (fc_stats) {
        unsigned long long h[3];
        FX_CUDA(cudaMemcpyAsync(h, stats.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        FX_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "fc_stats: objects %lld, all-class %llu, re-scored %llu, candidates %llu\n", (long long)n, h[0],
                h[1], h[2]);
    }
}

__global__ void k_dense_rowptrs(int64_t rows, int64_t row_bytes, const char *base, const char **out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < rows) out[i] = base + i * row_bytes;
}

void launch_rowptrs(int64_t rows, int64_t row_bytes, const char *base, const char **out, cudaStream_t st) {
    if (rows <= 0) return;
    k_dense_rowptrs<<<(unsigned)cdiv(rows, 256), 256, 0, st>>>(rows, row_bytes, base, out);
    FX_LAUNCHED();
}

void launch_row_norms(int64_t rows, int D, const float *X, float *out, cudaStream_t st) {
    if (rows <= 0) return;
    k_row_norms<<<(unsigned)cdiv(rows * 32, 256), 256, 0, st>>>(rows, D, X, out);
    FX_LAUNCHED();
}

}  // namespace fx
