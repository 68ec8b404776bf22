// screen_tc.cu -- K2a on the 5th-gen tensor cores: batch-object x snapshot-
// centroid squared distances via the GEMM expansion
//     d^2 = ||a||^2 + ||b||^2 - 2 a.b
// with a.b from tcgen05.mma kind::tf32 (A and B K-major in shared memory,
// accumulator in TMEM, 128 x 128 tile per CTA).
//
// Exactness: the screen only prunes.  Its rigorous error bound (consumed by
// tc_bounds in fx_internal.cuh) is
//     |a.b^ - a.b| <= gamma ||a|| ||b||,  gamma = 2^-9 + D 2^-22
// (TF32 keeps 10 mantissa bits of each operand, truncation or rounding:
// relative product error <= 2^-9 + 2^-20; plus the FP32 accumulation of D
// products), so d^2 lies within 2 gamma ||a|| ||b|| (+ FP32 rounding of the
// expansion) of the screen value.  The object's best candidate is then
// re-measured in FP32 direct-difference form (k_row_summary_tc), and every
// decision the bounds leave open goes to the exact float64 path.
//
// Operand staging: rows are gathered (batch objects through their feature row
// pointers, centroids through the snapshot slot list) with cp.async 16-byte
// copies into the canonical no-swizzle K-major layout: 8-row x 16-byte core
// matrices, K-adjacent core matrices 128 B apart (LBO), 8-row groups
// KT*32 B apart (SBO).  A 4-stage cp.async ring feeds the single MMA-issuing
// thread; tcgen05.commit on a per-stage mbarrier releases a stage.
#include <algorithm>
#include <cstdlib>
#include <string>

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "fx_handles.cuh"
#include "tc_common.cuh"

namespace cg = cooperative_groups;

namespace fx {

constexpr int TC_M = 128, TC_N = 128, TC_STAGES = 6, TC_STAGES2 = 3, TC_THREADS = 256;  // warps 4-7 only help load
constexpr int TC_TILE_BYTES = TC_M * TC_KT * 4;  // 16 KB per operand per stage

// Operand staging by TMA (TMA = true): one 2-D tiled box (32 fp32 x 128 rows,
// SWIZZLE_128B K-major: 8-row x 128 B atoms, 16-byte chunk c of row r at
// c ^ (r % 8)) per operand and stage.  A = consecutive feature rows of the
// ingest call (tmA): with compact features the batch's rows themselves, else
// the object rows spanning the batch, duplicates included -- rmap gives each
// object row's classified index (-1: duplicate, its outputs are dropped).
// B = the snapshot packed in snapshot order (tmB over C32q, k_snap_pack).
// One producer thread, one MMA-issuing thread, four warps that fold the row
// norms out of each stage; per-stage full barriers count bytes (expect_tx),
// empty barriers the MMA commit plus the four norm warps.

// out[a][q] = ||A_a||^2 + ||B_q||^2 - 2 A_a.B_q   (float, not clamped)
template <bool TMA, int ST>
__global__ void __launch_bounds__(TC_THREADS, 1) k_screen_tc(int nA, int64_t a0, const char *const *__restrict__ frow,
                                                           const float *fnorm, int D,  // aliases fnorm_out
                                                           const int64_t *__restrict__ nB_dev,
                                                           const float *__restrict__ C32,
                                                           const int32_t *__restrict__ snap,
                                                           const float *__restrict__ cn2, float *__restrict__ out,
                                                           int64_t ld, int kchunk, int dbg, float *__restrict__ fnorm_out,
                                                           ScreenModel sm, double T, int32_t *__restrict__ res_col,
                                                           int32_t *__restrict__ res_pos, int64_t *__restrict__ nres,
                                                           int *__restrict__ rowmin_g, float *__restrict__ snorm,
                                                           const __grid_constant__ CUtensorMap tmA,
                                                           const __grid_constant__ CUtensorMap tmB, int rbase, int nR,
                                                           const int32_t *__restrict__ rmap) {
    pdl_enter();
    // blockIdx.z selects the K range [z*kchunk, (z+1)*kchunk) (split-K when the
    // tile grid alone cannot fill the machine; partials are atomically added).
    // blockIdx.x = column tile * row tiles + row tile: the CTAs that share a
    // snapshot tile run back to back, so it streams from HBM once per batch.
    const int nB = (int)*nB_dev;
    // tile rows: batch rows (rmap == nullptr) or the object rows rbase.. of tmA
    const int nrt = (nR + TC_M - 1) / TC_M;
    const int tb = (int)(blockIdx.x / nrt) * TC_N, ta = (int)(blockIdx.x % nrt) * TC_M;
    auto row_cls = [&](int tr) {  // batch-local classified index of tile-space row tr, -1: none
        if (tr >= nR) return -1;
        if (!rmap) return tr < nA ? tr : -1;
        const int c = rmap[rbase + tr];
        return c >= 0 ? (int)(c - a0) : -1;
    };
    if (nB == 0 && tb == 0 && blockIdx.z == 0 && threadIdx.x < TC_M) {
        // empty snapshot (stream start): no screen, but the batch still needs ||f||
        const int a = row_cls(ta + threadIdx.x);
        if (a >= 0 && fnorm_out) {
            const float *row = (const float *)frow[a0 + a];
            float tot = 0.f;
            for (int k0 = 0; k0 < D; k0 += TC_KT) {
                float p = 0.f;
                for (int k = k0; k < min(D, k0 + TC_KT); k++) p = fmaf(row[k], row[k], p);
                tot += p;
            }
            fnorm_out[a0 + a] = sqrtf(tot);
        }
        if (a >= 0 && res_col) {  // no live cluster: every object is a probable seed
            const int col = (int)atomicAdd((unsigned long long *)nres, 1ull);
            res_pos[col] = a;
            res_col[a] = col;
        }
    }
    if (tb >= nB || ta >= nR || (dbg & 8)) return;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // [stage][A 16KB | B 16KB], 1024-byte aligned (SWIZZLE_128B atoms)
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ const float *rowsA[TC_M];
    __shared__ const float *rowsB[TC_N];
    __shared__ int rcls[TC_M];  // batch-local classified index of each tile row, -1: none
    __shared__ float cn2t[TC_N];  // ||c||^2 of the tile's snapshot columns (gathered once)
    __shared__ __align__(8) uint64_t bar_stage[ST];
    __shared__ __align__(8) uint64_t bar_full[ST];
    __shared__ __align__(8) uint64_t bar_done;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int r = tid; r < TC_M; r += TC_THREADS) {
        const int a = row_cls(ta + r);
        rcls[r] = a;
        cn2t[r] = tb + r < nB ? cn2[snap[tb + r]] : 0.f;
        if (!TMA) {
            const int b = tb + r;
            rowsA[r] = a >= 0 ? (const float *)frow[a0 + a] : nullptr;
            rowsB[r] = b < nB ? C32 + (int64_t)snap[b] * D : nullptr;
        }
    }
    if (tid == 0) {
        for (int s = 0; s < ST; s++) {
            mbar_init(&bar_stage[s], TMA ? 5 : 1);
            mbar_init(&bar_full[s], 1);
        }
        mbar_init(&bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "r"(TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    const uint32_t tmem = tmem_base;
    const uint32_t sbase = smem_u32(smem);

    const int kbeg = blockIdx.z * kchunk, kend = min(D, kbeg + kchunk);
    const int nk = kend > kbeg ? (kend - kbeg + TC_KT - 1) / TC_KT : 0;
    // instruction descriptor: D=F32, A=B=TF32, K-major both, N=128, M=128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                           ((uint32_t)(TC_M >> 4) << 24);
    float a2 = 0.f;  // ||A_row||^2 of this thread's row over the CTA's K range (fp32, per-stage partials)
    if (TMA) {
        if (warp == 4 && lane == 0) {  // producer: one 128-row box of A and of B per stage
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
            for (int it = 0; it < nk; it++) {
                const int s = it % ST;
                if (it >= ST) mbar_wait(&bar_stage[s], (uint32_t)(((it / ST) - 1) & 1));
                const uint32_t st = sbase + s * 2 * TC_TILE_BYTES;
                const uint32_t fb = smem_u32(&bar_full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(2 * TC_TILE_BYTES)
                             : "memory");
                const int k = kbeg + it * TC_KT;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3}], [%4];\n" ::"r"(st),
                    "l"(&tmA), "r"(k), "r"(rbase + ta), "r"(fb)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3}], [%4];\n" ::"r"(st + TC_TILE_BYTES),
                    "l"(&tmB), "r"(k), "r"(tb), "r"(fb)
                    : "memory");
            }
        } else if (warp == 5) {  // MMA issue
            for (int it = 0; it < nk; it++) {
                const int s = it % ST;
                mbar_wait(&bar_full[s], (uint32_t)((it / ST) & 1));
                if (lane == 0) {
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
                    const uint32_t st = sbase + s * 2 * TC_TILE_BYTES;
#pragma unroll
                    for (int kk = 0; kk < TC_KT / 8; kk++) {
                        const uint64_t da = umma_desc_sw128(st + kk * 32);
                        const uint64_t db = umma_desc_sw128(st + TC_TILE_BYTES + kk * 32);
                        const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                            "l"(da), "l"(db), "r"(idesc), "r"(acc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&bar_stage[s])));
                }
                __syncwarp();
            }
            if (lane == 0)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&bar_done)));
        } else if (warp < 4) {  // row norms: row tid's 8 chunks of 16 B in the swizzled atom
            for (int it = 0; it < nk; it++) {
                const int s = it % ST;
                mbar_wait(&bar_full[s], (uint32_t)((it / ST) & 1));
                const unsigned char *row = smem + s * 2 * TC_TILE_BYTES + (tid >> 3) * 1024 + (tid & 7) * 128;
                float p = 0.f;
#pragma unroll
                for (int c = 0; c < TC_KT / 4; c++) {
                    const float4 x = *(const float4 *)(row + ((c ^ (tid & 7)) << 4));
                    p = fmaf(x.x, x.x, p);
                    p = fmaf(x.y, x.y, p);
                    p = fmaf(x.z, x.z, p);
                    p = fmaf(x.w, x.w, p);
                }
                a2 += p;
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar_stage[s])));
            }
        }
    } else {
        auto kof = [&](int i) { return kbeg + i * TC_KT; };
        // prologue: stages 0..S-2
        for (int s = 0; s < ST - 1; s++) {
            if (s < nk && !(dbg & 1)) {
                const uint32_t st = sbase + s * 2 * TC_TILE_BYTES;
                load_tile<TC_M, TC_THREADS>(st, rowsA, kof(s), kend, fnorm);
                load_tile<TC_N, TC_THREADS>(st + TC_TILE_BYTES, rowsB, kof(s), kend, fnorm);
            }
            asm volatile("cp.async.commit_group;\n" ::);
        }
        for (int it = 0; it < nk; it++) {
            const int s = it % ST;
            asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2));
            asm volatile("fence.proxy.async.shared::cta;\n" ::);
            __syncthreads();
            if (tid < TC_M) {  // the row norm rides along: row tid's 32 values of this stage (stable until its refill)
                const unsigned char *stg = smem + s * 2 * TC_TILE_BYTES;
                float p = 0.f;
#pragma unroll
                for (int c = 0; c < TC_KT / 4; c++) {
                    const float4 x = *(const float4 *)(stg + ((((tid >> 3) * (TC_KT / 4) + c) << 7) + ((tid & 7) << 4)));
                    p = fmaf(x.x, x.x, p);
                    p = fmaf(x.y, x.y, p);
                    p = fmaf(x.z, x.z, p);
                    p = fmaf(x.w, x.w, p);
                }
                a2 += p;
            }
            if (tid == 0 && !(dbg & 2)) {
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
                const uint32_t st = sbase + s * 2 * TC_TILE_BYTES;
#pragma unroll
                for (int kk = 0; kk < TC_KT / 8; kk++) {
                    const uint64_t da = umma_desc(st + kk * 256, 128, TC_KT * 32);
                    const uint64_t db = umma_desc(st + TC_TILE_BYTES + kk * 256, 128, TC_KT * 32);
                    const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                        "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&bar_stage[s])));
            }
            // refill the stage consumed S-1 iterations from now
            const int nt = it + ST - 1;
            if (nt < nk) {
                const int ns = nt % ST;
                if (nt >= ST && !(dbg & 2)) mbar_wait(&bar_stage[ns], (uint32_t)(((nt / ST) - 1) & 1));
                const uint32_t st = sbase + ns * 2 * TC_TILE_BYTES;
                if (!(dbg & 1)) {
                    load_tile<TC_M, TC_THREADS>(st, rowsA, kof(nt), kend, fnorm);
                    load_tile<TC_N, TC_THREADS>(st + TC_TILE_BYTES, rowsB, kof(nt), kend, fnorm);
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        }
    }
    if (!TMA && tid == 0 && !(dbg & 2))
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&bar_done)));
    if (!(dbg & 2)) mbar_wait(&bar_done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    if (dbg & 4) {  // timing probe: no epilogue
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TC_N));
        return;
    }

    // epilogue: warp w owns TMEM lanes 32w..32w+31 = tile rows.  The partial
    // dot products go to a [128][TC_N+1] tile in this CTA's (now idle)
    // pipeline shared memory; the split-K CTAs of one output tile form a
    // thread-block cluster, and CTA rank z reduces rows z*128/split.. of the
    // tile over every CTA's shared memory (DSMEM, fixed order), adds the norms
    // and writes the rows coalesced.  No atomics, no pre-zeroed output.
    constexpr int TS = TC_N + 4;  // 16-byte aligned rows for the v4 DSMEM reads
    float *tile = (float *)smem;
    const int r = warp * 32 + lane;
    for (int c0 = 0; c0 < TC_N && warp < TC_M / 32; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
        for (int j = 0; j < 32; j++) tile[r * TS + c0 + j] = ((dbg & 2) || nk == 0) ? 0.f : __uint_as_float(v[j]);
    }
    if (warp < TC_M / 32) tile[r * TS + TC_N] = a2;
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    const int split = gridDim.z;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    const int rank = (int)cluster.block_rank();
    const int rows_per = (TC_M + split - 1) / split;
    const int r_lo = rank * rows_per, r_hi = min(TC_M, r_lo + rows_per);
    const int ncol = min(TC_N, nB - tb);
    const int nc4 = (ncol + 3) >> 2;
    const float *part[8];
#pragma unroll
    for (int q = 0; q < 8; q++) part[q] = q < split ? cluster.map_shared_rank(tile, q) : tile;
    __shared__ int rowmin[TC_M];  // min screen lower bound per row (non-negative float bits)
    for (int i = tid; i < TC_M; i += TC_THREADS) rowmin[i] = 0x7f800000;  // +inf
    __syncthreads();
    for (int e = tid; e < (r_hi - r_lo) * nc4; e += TC_THREADS) {
        const int rr = r_lo + e / nc4, c = (e % nc4) * 4;
        const int a = rcls[rr];
        if (a < 0) continue;
        float4 dot = make_float4(0.f, 0.f, 0.f, 0.f);
        float fa2 = 0.f;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (q < split) {
                const float4 x = *(const float4 *)(part[q] + rr * TS + c);
                dot.x += x.x;
                dot.y += x.y;
                dot.z += x.z;
                dot.w += x.w;
                fa2 += part[q][rr * TS + TC_N];
            }
        }
        if (c == 0 && fnorm_out) fnorm_out[a0 + a] = sqrtf(fa2);
        float *o = out + (int64_t)a * ld + tb + c;
        const float d4[4] = {dot.x, dot.y, dot.z, dot.w};
        float mn = INFINITY;
        const float fn = sqrtf(fa2);
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (c + j < ncol) {
                const float c2 = cn2t[c + j];
                const float v = fa2 + c2 - 2.f * d4[j];
                o[j] = v;
                if (res_col || rowmin_g) {
                    float lb, ub;
                    snap_bounds(sm, v, sqrtf(c2) * 1.00001f, fnorm_out ? fn : fnorm[a0 + a], lb, ub);
                    mn = fminf(mn, lb);
                }
            }
        if (res_col || rowmin_g) atomicMin(&rowmin[rr], __float_as_int(fmaxf(mn, 0.f)));
    }
    if (snorm && ta == 0 && rank == 0)
        for (int c = tid; c < ncol; c += TC_THREADS) snorm[tb + c] = sqrtf(cn2t[c]) * 1.00001f;
    if (rowmin_g) {
        // several column tiles: per-row minimum across CTAs (k_res_from_min flags the residuals)
        __syncthreads();
        for (int rr = r_lo + tid; rr < r_hi; rr += TC_THREADS)
            if (rcls[rr] >= 0) atomicMin(&rowmin_g[rcls[rr]], rowmin[rr]);
    } else if (res_col) {
        // fused residual detection (one column tile = the whole snapshot):
        // objects with no snapshot centroid whose lower bound is <= T
        __syncthreads();
        for (int rr = r_lo + tid; rr < r_hi; rr += TC_THREADS) {
            const int a = rcls[rr];
            if (a < 0) continue;
            if ((double)__int_as_float(rowmin[rr]) > T) {
                const int col = (int)atomicAdd((unsigned long long *)nres, 1ull);
                res_pos[col] = a;
                res_col[a] = col;
            } else {
                res_col[a] = -1;
            }
        }
    }
    cluster.sync();  // keep this CTA's shared memory alive until every CTA of the cluster has read it
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TC_N));
}

size_t screen_tc_smem(int stages) {
    // pipeline stages; the epilogue's [128][TC_N+4] tile reuses them
    const size_t pipe = (size_t)stages * 2 * TC_TILE_BYTES;
    return std::max(pipe, (size_t)TC_M * (TC_N + 4) * 4) + 1024;
}

// 2-D tensor map over fp32 rows for tile::gather4 (box 32 x 1, SWIZZLE_128B).
// False when the driver rejects it (alignment): the caller keeps cp.async.
bool make_rows_map(CUtensorMap *tm, const void *base, int64_t rows, int D, int64_t row_bytes, int box_rows) {
    static PFN_cuTensorMapEncodeTiled fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        if (!fn) return false;
    }
    if (rows <= 0 || ((uintptr_t)base & 15) || (row_bytes & 15)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {(cuuint32_t)TC_KT, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_screen_tc(int nA, int64_t a0, const char *const *frow, const float *fnorm, int D, const int64_t *nB_dev,
                      int nB_max, const float *C32, const int32_t *snap, const float *cn2, float *out, int64_t ld,
                      cudaStream_t st, float *fnorm_out, ScreenModel sm, double T, int32_t *res_col,
                      int32_t *res_pos, int64_t *nres, int *rowmin_g, float *snorm, const CUtensorMap *tmA,
                      const CUtensorMap *tmB, int rbase, int nR, const int32_t *rmap) {
    // residual detection inside one tile, or across tiles through rowmin_g
    if (nB_max > TC_N) res_col = nullptr;
    else rowmin_g = nullptr;
    static bool attr_set[64] = {};
    bool &attr = attr_set[dev_slot()];
    if (!attr) {
        for (auto k : {k_screen_tc<false, TC_STAGES>, k_screen_tc<true, TC_STAGES>})
            FX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)screen_tc_smem(TC_STAGES)));
        FX_CUDA(cudaFuncSetAttribute(k_screen_tc<true, TC_STAGES2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)screen_tc_smem(TC_STAGES2)));
        attr = true;
    }
    const bool tma = tmA && tmB;
    static const CUtensorMap zero_map = {};
    static const int dbg = getenv("FOCUS_B200_TCDBG") ? atoi(getenv("FOCUS_B200_TCDBG")) : 0;
    static const int split_env = getenv("FOCUS_B200_TCSPLIT") ? atoi(getenv("FOCUS_B200_TCSPLIT")) : 0;
    if (!tma) {  // cp.async staging gathers the batch rows themselves
        rbase = 0;
        nR = nA;
        rmap = nullptr;
    }
    const int64_t tiles = cdiv(nB_max, TC_N) * cdiv(nR, TC_M);
    // split-K: the largest factor that keeps the grid in one wave (one CTA
    // per SM) with >= 4 pipeline stages per CTA
    int split = 1;
    while (split < 8 && tiles * (split + 1) <= 148 && D / (split + 1) >= 4 * TC_KT) split++;
    // FOCUS_B200_TC2=1: two CTAs per SM (TC_STAGES2-stage rings, 97 KB each)
    // when a 2-way split no longer fits one CTA per SM but fits two.  Measured
    // at C2 (B = 8192, 80 row tiles -> 160 CTAs): screen 42.8 -> 39.3 us per
    // launch, but the stream is not faster (44.4 vs 44.8 M objects/s, one run
    // of four stalled at 32.7 M): the half-SM CTAs delay the PDL-launched
    // kernels behind them.  Off by default.
    static const bool two_env = getenv("FOCUS_B200_TC2") && atoi(getenv("FOCUS_B200_TC2")) == 1;
    bool two = false;
    if (tma && two_env && split == 1 && tiles * 2 > 148 && tiles * 2 <= 2 * 148 && D / 2 >= 4 * TC_KT) {
        split = 2;
        two = true;
    }
    if (split_env > 0) split = split_env;
    split = std::min(split, 8);  // split-K CTAs of a tile form one (portable-size) cluster
    const int kchunk = (int)(cdiv(cdiv(D, split), TC_KT) * TC_KT);
    split = (int)cdiv(D, kchunk);  // no empty K range
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(cdiv(nB_max, TC_N) * cdiv(nR, TC_M)), 1, (unsigned)split);
    lc.blockDim = dim3(TC_THREADS);
    lc.dynamicSmemBytes = screen_tc_smem(two ? TC_STAGES2 : TC_STAGES);
    lc.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = (unsigned)split;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: see pdl_enter
    at[1].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl_enabled() ? 2 : 1;
    FX_CUDA(cudaLaunchKernelEx(&lc,
                               two   ? k_screen_tc<true, TC_STAGES2>
                               : tma ? k_screen_tc<true, TC_STAGES>
                                     : k_screen_tc<false, TC_STAGES>,
                               nA, a0, frow, fnorm, D, nB_dev, C32,
                               snap, cn2, out, ld, kchunk, dbg, fnorm_out, sm, T, res_col, res_pos, nres, rowmin_g,
                               snorm, tma ? *tmA : zero_map, tma ? *tmB : zero_map, rbase, nR, rmap));
    FX_LAUNCHED();
}

__global__ void k_rowptrs(int64_t n, const float *base, int dim, const char **rows, float *norm2) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    rows[i] = (const char *)(base + i * dim);
    float acc = 0.f;
    for (int k = 0; k < dim; k++) acc = fmaf(base[i * dim + k], base[i * dim + k], acc);
    norm2[i] = acc;
}
__global__ void k_iota32(int64_t n, int32_t *o) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) o[i] = (int32_t)i;
}
__global__ void k_sqrt_inplace(int64_t n, float *x) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = sqrtf(x[i]);
}

}  // namespace fx

extern "C" int fx_debug_screen_tc(int32_t device, int64_t na, int64_t nb, int32_t dim, const float *A, const float *B,
                                  float *out) {
    using namespace fx;
    try {
        if (dim % 4 != 0 || na <= 0 || nb <= 0) throw Error{FX_E_USAGE, "bad shapes"};
        FX_CUDA(cudaSetDevice(device));
        cudaStream_t st = 0;
        DevBuf<float> dA, dB, nA2, nB2, dout;
        DevBuf<const char *> rows;
        DevBuf<int32_t> snap;
        DevBuf<int64_t> nbd;
        dA.reserve((size_t)na * dim);
        dB.reserve((size_t)nb * dim);
        nA2.reserve(na);
        nB2.reserve(nb);
        dout.reserve((size_t)na * nb);
        rows.reserve(na);
        snap.reserve(nb);
        nbd.reserve(1);
        FX_CUDA(cudaMemcpy(dA.p, A, sizeof(float) * na * dim, cudaMemcpyHostToDevice));
        FX_CUDA(cudaMemcpy(dB.p, B, sizeof(float) * nb * dim, cudaMemcpyHostToDevice));
        FX_CUDA(cudaMemcpy(nbd.p, &nb, sizeof(int64_t), cudaMemcpyHostToDevice));
        DevBuf<const char *> rowsB;
        rowsB.reserve(nb);
        k_rowptrs<<<(unsigned)cdiv(na, 256), 256>>>(na, dA.p, dim, rows.p, nA2.p);
        k_rowptrs<<<(unsigned)cdiv(nb, 256), 256>>>(nb, dB.p, dim, rowsB.p, nB2.p);
        k_iota32<<<(unsigned)cdiv(nb, 256), 256>>>(nb, snap.p);
        k_sqrt_inplace<<<(unsigned)cdiv(na, 256), 256>>>(na, nA2.p);  // fnorm = ||a||
        FX_LAUNCHED();
        CUtensorMap tmA, tmB;
        const char *mode = getenv("FOCUS_B200_TCLOAD");
        const bool tma = !(mode && std::string(mode) == "cp") &&
                         make_rows_map(&tmA, dA.p, na, dim, (int64_t)dim * 4, TC_M) &&
                         make_rows_map(&tmB, dB.p, nb, dim, (int64_t)dim * 4, TC_N);
        launch_screen_tc((int)na, 0, rows.p, nA2.p, dim, nbd.p, (int)nb, dB.p, snap.p, nB2.p, dout.p, nb, st, nullptr,
                         ScreenModel{}, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, tma ? &tmA : nullptr,
                         tma ? &tmB : nullptr, 0, (int)na, nullptr);
        FX_CUDA(cudaDeviceSynchronize());
        FX_CUDA(cudaMemcpy(out, dout.p, sizeof(float) * na * nb, cudaMemcpyDeviceToHost));
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    }
    return FX_OK;
}
