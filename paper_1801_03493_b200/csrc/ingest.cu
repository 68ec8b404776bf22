// ingest.cu -- K0 pixel differencing, K1a rank-model top-K, K2 clustering
// (screen / resolve / fold), deferred seal.  SURVEY.md §2 kernel set.
//
// Reference semantics (clustering.py:86-160, ingest.py:50-96):
//   * objects are processed in stream order; a classified object joins the
//     live cluster with the smallest float64 distance (first minimum = smallest
//     cluster id) iff that distance <= T, else seeds a new cluster;
//   * after a seed, if more than M clusters are live, the live cluster with
//     the fewest members (dedup members included; ties -> smallest id) is
//     evicted;
//   * centroid = float64 running sum / featured count; representative =
//     featured member nearest the final centroid (ties -> first).
//
// B200 design: a batch of B classified objects is screened
// against the batch-start snapshot of the live centroids in FP32 with a
// rigorous error bound (k_screen); a single persistent CTA (k_resolve) then
// walks the batch in stream order keeping the exact sequential semantics:
// decisions that the bounds make certain cost O(L/threads) scalar work, the
// rest are decided by exact float64 distances (numpy pairwise order) against
// centroids materialised from the exact running sums.  k_fold then applies
// the batch's members to the float64 sums in order and refreshes the FP32
// snapshot.  Seal (representatives) is deferred to finalize, exactly as the
// reference's frozen-at-eviction centroids allow.
#include <chrono>
#include <climits>

#include "fx_handles.cuh"

namespace fx {

// ---------------------------------------------------------------------------
// K0: pixel differencing (ingest.py:37-47)
// ---------------------------------------------------------------------------

// K0: pixel_diff of every object against its predecessor (ingest.py:37-47).
// A CTA stages its 256 objects' signatures plus the predecessor's in shared
// memory with coalesced loads (row stride S + 1 doubles: conflict-free
// column reads), then each thread takes numpy's pairwise mean of |a - b|.
constexpr int DUP_T = 256, DUP_SMAX = 20;
__global__ void __launch_bounds__(DUP_T) k_dup_flags(int64_t n, int S, const int64_t *__restrict__ fid,
                                                     const double *__restrict__ sig, int has_prev, int64_t prev_fid,
                                                     const double *__restrict__ prev_sig, double eps,
                                                     uint8_t *__restrict__ is_dup) {
    __shared__ double ssig[(DUP_T + 1) * (DUP_SMAX + 1)];
    const int64_t i0 = (int64_t)blockIdx.x * DUP_T;
    const int tid = threadIdx.x;
    const int64_t i = i0 + tid;
    const bool staged = S <= DUP_SMAX;
    if (staged && eps >= 0.0) {
        const int64_t rem = n - i0 + 1;
        const int nrow = (int)(rem < DUP_T + 1 ? rem : DUP_T + 1);  // rows i0-1 .. i0+DUP_T-1
        for (int e = tid; e < nrow * S; e += DUP_T) {
            const int r = e / S, k = e % S;
            const int64_t src = i0 - 1 + r;
            double v = 0.0;
            if (src >= 0) v = sig[src * S + k];
            else if (has_prev) v = prev_sig[k];
            ssig[r * (S + 1) + k] = v;
        }
    }
    __syncthreads();
    if (i >= n) return;
    uint8_t d = 0;
    if (eps >= 0.0) {
        int64_t pf = 0;
        bool have = false;
        if (i > 0) {
            pf = fid[i - 1];
            have = true;
        } else if (has_prev) {
            pf = prev_fid;
            have = true;
        }
        if (have && fid[i] - pf <= 1) {
            double sum;
            if (staged) {
                const double *a = ssig + tid * (S + 1), *b = ssig + (tid + 1) * (S + 1);
                sum = pw_sum_seq(S, [&](int k) { return fabs(dsub(a[k], b[k])); });
            } else {
                const double *a = i > 0 ? sig + (i - 1) * S : prev_sig;
                const double *b = sig + i * S;
                sum = pw_sum_seq(S, [&](int k) { return fabs(dsub(a[k], b[k])); });
            }
            d = ddiv(sum, (double)S) <= eps;
        }
    }
    is_dup[i] = d;
}

// classified-object bookkeeping: cls index, feature row pointer, dup runs
__global__ void k_compact_cls(int64_t n, int64_t obj_base, int64_t cls_base, const uint8_t *__restrict__ is_dup,
                              const int64_t *__restrict__ excl, const char *feat_base, int64_t row_bytes,
                              int compact, int64_t *__restrict__ cls_obj, const char **__restrict__ frow,
                              int32_t *__restrict__ dup_run, int32_t *__restrict__ orow) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t e = excl[i];
    if (orow) orow[i] = is_dup[i] ? -1 : (int32_t)(cls_base + e);  // object row -> classified index
    if (!is_dup[i]) {
        int64_t c = cls_base + e;
        cls_obj[c] = obj_base + i;
        frow[c] = feat_base + (compact ? e : i) * row_bytes;
        dup_run[c] = 0;
    }
}

__global__ void k_dup_runs(int64_t n, int64_t cls_base, const uint8_t *__restrict__ is_dup,
                           const int64_t *__restrict__ excl, int32_t *__restrict__ dup_run) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (is_dup[i]) atomicAdd(&dup_run[cls_base + excl[i] - 1], 1);
}

template <typename T>
__global__ void k_fnorm(int64_t c0, int64_t nc, int D, const char *const *__restrict__ frow, float *__restrict__ fnorm) {
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (w >= nc) return;
    const T *f = (const T *)frow[c0 + w];
    float acc = 0.f;
    for (int k = lane; k < D; k += 32) {
        float x = (float)f[k];
        acc = fmaf(x, x, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) fnorm[c0 + w] = sqrtf(acc);
}

// ---------------------------------------------------------------------------
// K1a: rank-model top-K (classifiers.py:126-149, core.py:60-61)
// ---------------------------------------------------------------------------

__global__ void k_rank_topk(int64_t c0, int64_t nc, const int64_t *__restrict__ cls_obj, const int64_t *__restrict__ oid,
                            const int32_t *__restrict__ tcls, int K, int V, int gt, uint64_t seed,
                            const uint64_t *__restrict__ thr, const int32_t *__restrict__ emit,
                            const int32_t *__restrict__ fill, int32_t *__restrict__ topk,
                            unsigned long long *__restrict__ err_obj) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nc) return;
    int64_t obj = cls_obj[c0 + i];
    int c = tcls[obj];
    if (c < 0 || c >= V) {  // unlabeled: MissingTrueClass raised lazily (classifiers.py:128-129)
        atomicMin(err_obj, (unsigned long long)obj);
        return;
    }
    int rank = 1;
    if (!gt) {
        uint64_t u = first_u53(seed, (uint64_t)oid[obj], 0ull);
        for (int j = 0; j < K; j++) rank += thr[j] <= u;
    }
    int e = emit[c];
    const int32_t *row = fill + (int64_t)e * K;
    int32_t *out = topk + obj * K;
    for (int j = 0; j < K; j++) out[j] = j < rank - 1 ? row[j] : (j == rank - 1 ? e : row[j - 1]);
}

// ---------------------------------------------------------------------------
// K2a: FP32 distance screen (direct difference, two-level accumulation)
//   dist[a][b] = sqrt(sum_k (A_a[k] - B_b[k])^2), 64x64 tile / CTA.
// Error model: relative error of the squared distance is
// <= (3 + 64 + ceil(D/64) + 2) * 2^-24 -- every 64 dims the running partial is
// flushed into the total.
// ---------------------------------------------------------------------------

constexpr int SC_T = 64, SC_K = 32;

template <typename TA, typename FB>
__global__ void __launch_bounds__(256) k_screen(int nA, int64_t a0, const char *const *__restrict__ frow, int D,
                                               const int64_t *__restrict__ nB_dev, int nB_max, FB fb,
                                               float *__restrict__ out, int64_t ld, int nB_skip = -1) {
    pdl_enter();
    const int nB = nB_dev ? (int)*nB_dev : nB_max;
    if (nB <= nB_skip) return;  // few residual columns: k_res_cols handles them
    // persistent over the (column, row) tiles that exist for the device-side nB
    const int ncol = (nB + SC_T - 1) / SC_T, nrow = (nA + SC_T - 1) / SC_T;
    for (int tile = blockIdx.x; tile < ncol * nrow; tile += gridDim.x) {
    const int tb = (tile % ncol) * SC_T, ta = (tile / ncol) * SC_T;
    __shared__ float As[SC_K][SC_T + 1];
    __shared__ float Bs[SC_K][SC_T + 1];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    float acc[4][4], tot[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = tot[i][j] = 0.f;
    for (int k0 = 0; k0 < D; k0 += SC_K) {
#pragma unroll
        for (int e = 0; e < 8; e++) {
            int idx = tid + e * 256, r = idx >> 5, k = idx & 31;
            float va = 0.f, vb = 0.f;
            if (ta + r < nA && k0 + k < D) va = (float)((const TA *)frow[a0 + ta + r])[k0 + k];
            if (tb + r < nB && k0 + k < D) vb = fb(tb + r, k0 + k);
            As[k][r] = va;
            Bs[k][r] = vb;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < SC_K; k++) {
            float ra[4], rb[4];
#pragma unroll
            for (int i = 0; i < 4; i++) ra[i] = As[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; j++) rb[j] = Bs[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    float d = ra[i] - rb[j];
                    acc[i][j] = fmaf(d, d, acc[i][j]);
                }
        }
        __syncthreads();
        if (((k0 / SC_K) & 1) || k0 + SC_K >= D) {
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    tot[i][j] += acc[i][j];
                    acc[i][j] = 0.f;
                }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        int a = ta + ty * 4 + i;
        if (a >= nA) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int b = tb + tx * 4 + j;
            if (b < nB) out[(int64_t)a * ld + b] = sqrtf(tot[i][j]);
        }
    }
    __syncthreads();
    }
}

struct FromSnapshot {  // B rows = FP32 snapshot centroids of the live slots
    const float *C32;
    const int32_t *snap;
    int D;
    __device__ float operator()(int b, int k) const { return C32[(int64_t)snap[b] * D + k]; }
};
template <typename T>
struct FromResidual {  // B rows = features of the batch's residual objects
    const char *const *frow;
    int64_t a0;
    const int32_t *res_pos;
    __device__ float operator()(int b, int k) const { return (float)((const T *)frow[a0 + res_pos[b]])[k]; }
};

// residual detection: object has no snapshot centroid whose screen lower
// bound is <= T -> it will very likely seed; its column of object-object
// distances is precomputed for the objects after it.
__global__ void k_residuals(int nA, const int64_t *__restrict__ ctr, const float *__restrict__ dist, int64_t ld,
                            const float *__restrict__ cn2, const int32_t *__restrict__ snap,
                            const float *__restrict__ fnorm, int64_t a0, ScreenModel sm, double T,
                            int32_t *__restrict__ res_col, int32_t *__restrict__ res_pos, int64_t *__restrict__ nres) {
    pdl_enter();
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= nA) return;
    const int nsnap = (int)ctr[C_NSNAP];
    const float fn = fnorm[a0 + w];
    float mn = INFINITY;
    for (int q = lane; q < nsnap; q += 32) {
        float lb, ub;
        snap_bounds(sm, dist[(int64_t)w * ld + q], sqrtf(cn2[snap[q]]) * 1.00001f, fn, lb, ub);
        mn = fminf(mn, lb);
    }
    mn = warp_min(mn);
    if (lane == 0) {
        if ((double)mn > T) {
            int col = (int)atomicAdd((unsigned long long *)nres, 1ull);
            res_pos[col] = w;
            res_col[w] = col;
        } else {
            res_col[w] = -1;
        }
    }
}

// Residual columns when there are few of them (the common case: a batch has
// 0..a handful of probable seeds).  dres[b][col] = FP32 direct-difference
// distance between object b and residual `col`, needed only for b after the
// residual's own position (the seed can only influence later objects).  One
// warp per row; the residual rows are staged in shared memory RC_COLS at a
// time.  Error model: each lane sums D/32 squared differences, flushing its
// running partial every 64 terms, then a 5-level warp tree -- within the
// SIMT screen model of screen_rel(D) for every D.
constexpr int RC_MAX = 64, RC_COLS = 8;

template <typename T>
__global__ void __launch_bounds__(256) k_res_cols(int nA, int64_t a0, const char *const *__restrict__ frow, int D,
                                                 const int64_t *__restrict__ nres_dev,
                                                 const int32_t *__restrict__ res_pos, float *__restrict__ out,
                                                 int64_t ld) {
    const int nres = (int)*nres_dev;
    if (nres == 0 || nres > RC_MAX) return;
    extern __shared__ float rc_s[];  // [RC_COLS][D]
    __shared__ int s_pos[RC_COLS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int cc = 0; cc < nres; cc += RC_COLS) {
        const int ncol = min(RC_COLS, nres - cc);
        __syncthreads();
        if (threadIdx.x < RC_COLS) s_pos[threadIdx.x] = threadIdx.x < ncol ? res_pos[cc + threadIdx.x] : INT_MAX;
        for (int e = threadIdx.x; e < ncol * D; e += blockDim.x) {
            const int j = e / D, k = e - j * D;
            rc_s[e] = (float)((const T *)frow[a0 + res_pos[cc + j]])[k];
        }
        __syncthreads();
        int pmin = INT_MAX;
#pragma unroll
        for (int j = 0; j < RC_COLS; j++) pmin = min(pmin, s_pos[j]);
        for (int b = pmin + 1 + blockIdx.x * nw + wid; b < nA; b += gridDim.x * nw) {
            const T *f = (const T *)frow[a0 + b];
            float tot[RC_COLS], acc[RC_COLS];
#pragma unroll
            for (int j = 0; j < RC_COLS; j++) tot[j] = acc[j] = 0.f;
            int cnt = 0;
            for (int k = lane; k < D; k += 32) {
                const float x = (float)f[k];
#pragma unroll
                for (int j = 0; j < RC_COLS; j++) {
                    const float d = x - rc_s[j * D + k];
                    acc[j] = fmaf(d, d, acc[j]);
                }
                if (++cnt == 64) {
#pragma unroll
                    for (int j = 0; j < RC_COLS; j++) {
                        tot[j] += acc[j];
                        acc[j] = 0.f;
                    }
                    cnt = 0;
                }
            }
#pragma unroll
            for (int j = 0; j < RC_COLS; j++) {
                const float v = warp_sum(tot[j] + acc[j]);
                if (lane == j && j < ncol && b > s_pos[j]) out[(int64_t)b * ld + cc + j] = sqrtf(v);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K2b: sequential resolve (one CTA per stream per batch)
// ---------------------------------------------------------------------------

struct ResolveArgs {
    int B, Bcap;
    int64_t c0;
    int D;
    double T;
    int64_t M;
    float rel, absc;
    ScreenModel sm;
    const float *dist;
    int64_t ld;
    const float *dres;
    int64_t ldr;
    const int32_t *res_col, *res_pos;
    float *dod;
    const char *const *frow;
    const float *fnorm;
    const int32_t *dup_run;
    const int64_t *cls_obj;
    double *S;
    int32_t *s_cid, *s_nfeat, *s_size, *s_snapq, *s_seedpos, *s_foldpos, *s_pend, *s_odcol, *s_evicted, *s_didx;
    double *s_drift;
    float *s_cn2;
    int32_t *live, *live_pos, *free_stack, *defer_free, *snap_slot;
    int64_t *ctr;
    int32_t *slot_of, *pend_rank, *evict_slot, *evict_cid, *dirty, *dirty_off, *pend_list;
    int32_t *pend_seg;  // [B] dirty index of each pend_list entry
    int32_t *cid_slot, *s_fjoin, *ev_pos, *ev_vic;  // eviction FIFO: slot of each cid, first join, plan
    int32_t *cluster_of, *mrank, *frank;
    const PwPlan *plan;
    int32_t *s_grp;
    long long *prof;  // [16] cycles: A, B1B2, CD, confirm, E, seq; [6] windows, [7] seq steps; [8..15] confirms by batch bucket
    int batch_no;
    const int32_t *sum_slot, *sum_q;
    const float *sum_d1, *sum_e1, *sum_lbr;
    int64_t *h_ring;  // pinned host slot (UVA): counters the host reads two batches later
    const double *s_sdev;  // per slot: bound on |snapshot centroid - exact centroid| (k_tfold)
    // fast path scratch (k_rfast1 / k_rfast3)
    int32_t *f_rank, *f_dup, *f_ccnt, *f_cdup, *f_gi;
    float *f_P, *f_csum, *f_cmax, *f_gf;
    double *f_gd;
    unsigned char *rs_gobj;  // per-object state in global memory (B > 4096), else nullptr
    const unsigned long long *chain_epoch;  // lagged exact chains completed (k_fold's last CTA)
};

constexpr int RS_THREADS = 512;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_MAXCAND = 512;

struct Cand {
    float ub;
    int ubi;
    float lb1;
    int lb1i;
    float lb2;
};

__device__ __forceinline__ void cand_merge(Cand &a, const Cand &b) {
    if (b.ub < a.ub || (b.ub == a.ub && b.ubi < a.ubi)) {
        a.ub = b.ub;
        a.ubi = b.ubi;
    }
    // two smallest LBs
    if (b.lb1 < a.lb1) {
        a.lb2 = fminf(a.lb1, b.lb2);
        a.lb1 = b.lb1;
        a.lb1i = b.lb1i;
    } else {
        a.lb2 = fminf(a.lb2, b.lb1);
    }
}

template <typename T>
__device__ __forceinline__ void slot_bounds(const ResolveArgs &A, int b, float fn, int slot, float &lb, float &ub, float &d) {
    int q = A.s_snapq[slot];
    float cn;
    if (q >= 0) {
        const float v = A.dist[(int64_t)b * A.ld + q];
        cn = sqrtf(A.s_cn2[slot]) * 1.00001f;
        float l0, u0;
        snap_bounds(A.sm, v, cn, fn, l0, u0);
        d = 0.5f * (l0 + u0);
        const float dr = (float)A.s_drift[slot] * 1.00001f;
        lb = l0 - dr;
        ub = u0 + dr;
        lb = lb - fabsf(lb) * 1e-6f - 1e-30f;
        ub = ub + fabsf(ub) * 1e-6f + 1e-30f;
        return;
    } else {
        int s = A.s_seedpos[slot];
        int col = A.res_col[s];
        d = col >= 0 ? A.dres[(int64_t)b * A.ldr + col] : A.dod[(int64_t)A.s_odcol[slot] * A.B + b];
        cn = A.fnorm[A.c0 + s];
    }
    float e = A.rel * d + A.absc * (cn + fn) + 1e-30f;
    float dr = (float)A.s_drift[slot] * 1.00001f;
    lb = d - e - dr;
    ub = d + e + dr;
    // round the bounds outward (fp32 arithmetic of the bound itself)
    lb = lb - fabsf(lb) * 1e-6f - 1e-30f;
    ub = ub + fabsf(ub) * 1e-6f + 1e-30f;
}

// exact ||c_slot - f_b|| for the current centroid of `slot`: first fold the
// slot's in-batch members in [foldpos, b) into its float64 sum (stream
// order), then evaluate sqrt(pairwise_sum(((S/n) - f)^2)) in numpy's order.
template <typename T>
__device__ double exact_dist(const ResolveArgs &A, int b, int slot, const int32_t *sh_slot_of, int *mlist,
                             double *scratch, int nfeat = -1) {
    const int D = A.D;
    int fp = A.s_foldpos[slot];
    const int sp = A.s_seedpos[slot];
    double *Sj = A.S + (int64_t)slot * D;
    if (fp < b) {
        __shared__ int s_nm;
        if (threadIdx.x < 32) {
            int base = 0;
            for (int p0 = fp; p0 < b; p0 += 32) {
                int p = p0 + (int)threadIdx.x;
                bool hit = p < b && sh_slot_of[p] == slot;
                unsigned m = __ballot_sync(0xffffffffu, hit);
                if (hit) mlist[base + __popc(m & ((1u << threadIdx.x) - 1u))] = p;
                base += __popc(m);
            }
            if (threadIdx.x == 0) s_nm = base;
        }
        __syncthreads();
        const int nm = s_nm;
        const bool fresh = sp >= fp;  // seeded inside [fp, b): the seed row starts the sum
        for (int k = threadIdx.x; k < D; k += blockDim.x) {
            double s = fresh ? -0.0 : Sj[k];
            for (int i = 0; i < nm; i++) {
                const int p = mlist[i];
                double f = to_d(((const T *)A.frow[A.c0 + p])[k]);
                s = (p == sp) ? f : dadd(s, f);
            }
            Sj[k] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) A.s_foldpos[slot] = b;
    }
    const double n = (double)(nfeat >= 0 ? nfeat : A.s_nfeat[slot]);
    const T *f = (const T *)A.frow[A.c0 + b];
    __syncthreads();
    auto term = [&](int k) {
        double x = dsub(ddiv(Sj[k], n), to_d(f[k]));
        return dmul(x, x);
    };
    const PwPlan &P = *A.plan;
    double *chain = scratch, *node = scratch + P.n_chains;
    for (int c = threadIdx.x; c < P.n_chains; c += blockDim.x) {
        int lo = 0, hi = P.n_leaves - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (P.leaf_chain0[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const int s = P.leaf_start[lo], len = P.leaf_len[lo];
        double r;
        if (len < 8) {
            r = 0.0;
            for (int i = 0; i < len; i++) r = dadd(r, term(s + i));
        } else {
            const int a = c - P.leaf_chain0[lo], end = len - (len % 8);
            r = term(s + a);
            for (int i = 8 + a; i < end; i += 8) r = dadd(r, term(s + i));
        }
        chain[c] = r;
    }
    __syncthreads();
    for (int L = threadIdx.x; L < P.n_leaves; L += blockDim.x) {
        const int c0 = P.leaf_chain0[L], s = P.leaf_start[L], len = P.leaf_len[L];
        double res;
        if (len < 8) {
            res = chain[c0];
        } else {
            const double *r = chain + c0;
            res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
            for (int i = len - (len % 8); i < len; i++) res = dadd(res, term(s + i));
        }
        node[L] = res;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int o = 0; o < P.n_ops; o++) node[P.n_leaves + o] = dadd(node[P.op_left[o]], node[P.op_right[o]]);
    }
    __syncthreads();
    double tot = P.n_ops ? node[P.n_leaves + P.n_ops - 1] : node[0];
    __syncthreads();
    return __dsqrt_rn(dadd(0.0, tot));
}

// Scan of one screen row (one warp): best snapshot candidate by upper bound
// (ties: lower snapshot index), its interval, min lower bound of the rest.
// U loads per lane in flight; snorm (written by the TC screen) replaces the
// two-level gather cn2[snap[q]] when present.
__device__ __forceinline__ void row_scan(const float *__restrict__ drow, int nsnap, const float *__restrict__ cn2,
                                         const int32_t *__restrict__ snap, const float *__restrict__ snorm,
                                         ScreenModel sm, float fn, int lane, float &u1, float &l1, float &lbr, int &q1,
                                         int qbeg = 0) {
    constexpr int U = 8;
    u1 = INFINITY;
    l1 = INFINITY;
    lbr = INFINITY;
    q1 = -1;
    for (int q0 = qbeg; q0 < nsnap; q0 += 32 * U) {
        float dv[U], nv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int q = q0 + lane + 32 * u;
            dv[u] = q < nsnap ? drow[q] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int q = q0 + lane + 32 * u;
            nv[u] = q < nsnap ? (snorm ? snorm[q] : sqrtf(cn2[snap[q]]) * 1.00001f) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int q = q0 + lane + 32 * u;
            if (q < nsnap) {
                float lb, ub;
                snap_bounds(sm, dv[u], nv[u], fn, lb, ub);
                if (ub < u1) {
                    if (q1 >= 0) lbr = fminf(lbr, l1);
                    u1 = ub;
                    l1 = lb;
                    q1 = q;
                } else {
                    lbr = fminf(lbr, lb);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float ou = __shfl_xor_sync(0xffffffffu, u1, o), ol = __shfl_xor_sync(0xffffffffu, l1, o);
        const float olbr = __shfl_xor_sync(0xffffffffu, lbr, o);
        const int oq = __shfl_xor_sync(0xffffffffu, q1, o);
        const bool take = oq >= 0 && (q1 < 0 || ou < u1 || (ou == u1 && oq < q1));
        if (take) {
            lbr = fminf(fminf(lbr, olbr), q1 >= 0 ? l1 : INFINITY);
            u1 = ou;
            l1 = ol;
            q1 = oq;
        } else {
            lbr = fminf(fminf(lbr, olbr), oq >= 0 ? ol : INFINITY);
        }
    }
}

// Residual flags from the per-row minimum screen lower bound the multi-tile TC
// screen accumulated in rowmin (float bits); resets rowmin for the next batch.
__global__ void k_res_from_min(int nA, int *__restrict__ rowmin, double T, int32_t *__restrict__ res_col,
                               int32_t *__restrict__ res_pos, int64_t *__restrict__ nres) {
    pdl_enter();
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nA) return;
    const float mn = __int_as_float(rowmin[a]);
    rowmin[a] = 0x7f7f7f7f;
    if ((double)mn > T) {
        const int col = (int)atomicAdd((unsigned long long *)nres, 1ull);
        res_pos[col] = a;
        res_col[a] = col;
    } else {
        res_col[a] = -1;
    }
}

// Per-object summary of the snapshot screen row: best snapshot slot, its
// distance and error bound, and min over the other snapshot slots of
// (d - e).  One warp per object.
template <typename T>
__global__ void k_row_summary(int nA, const int64_t *__restrict__ ctr, const float *__restrict__ dist, int64_t ld,
                              const float *__restrict__ cn2, const int32_t *__restrict__ snap,
                              const float *__restrict__ fnorm, int64_t a0, ScreenModel sm, float rel, float absc,
                              const char *const *__restrict__ frow, const float *__restrict__ C32, int D,
                              int32_t *__restrict__ sum_slot, int32_t *__restrict__ sum_q, float *__restrict__ sum_d1,
                              float *__restrict__ sum_e1, float *__restrict__ sum_lbr,
                              const float *__restrict__ snorm) {
    pdl_enter();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= nA) return;
    const int nsnap = (int)ctr[C_NSNAP];
    const float fn = fnorm[a0 + w];
    // best candidate = smallest upper bound; lbr = min lower bound of the rest
    float u1, l1, lbr;
    int q1;
    row_scan(dist + (int64_t)w * ld, nsnap, cn2, snap, snorm, sm, fn, lane, u1, l1, lbr, q1);
    float d1 = 0.5f * (l1 + u1), e1 = 0.5f * (u1 - l1);
    if (sm.tc && q1 >= 0) {
        // re-measure the best candidate in FP32 direct-difference form (tight SIMT bound)
        const T *f = (const T *)frow[a0 + w];
        const float *c = C32 + (int64_t)snap[q1] * D;
        float tot = 0.f, acc = 0.f;
        int cnt = 0;
        for (int k = lane; k < D; k += 32) {
            const float d = (float)f[k] - c[k];
            acc = fmaf(d, d, acc);
            if (++cnt == 64) {
                tot += acc;
                acc = 0.f;
                cnt = 0;
            }
        }
        tot += acc;
        tot = warp_sum(tot);
        const float dd = sqrtf(tot);
        const float ee = rel * dd + absc * (sqrtf(cn2[snap[q1]]) * 1.00001f + fn) + 1e-30f;
        if (dd + ee < u1) {  // keep whichever interval is tighter (both are valid)
            d1 = dd;
            e1 = ee;
        }
    }
    if (lane == 0) {
        sum_slot[w] = q1 >= 0 ? snap[q1] : -1;
        sum_q[w] = q1;
        sum_d1[w] = d1;
        sum_e1[w] = e1;
        sum_lbr[w] = lbr;
    }
}


// Fused per-row pass for FP32 features with D % 4 == 0, D <= 128 * NV and
// 16-byte aligned rows (one warp per batch object, row held in registers as
// NV float4 per lane, lane l owning elements 4 (l + 32 j) .. +3):
//   * row summary of the snapshot screen (best candidate by upper bound, its
//     interval, min lower bound of the rest), as k_row_summary;
//   * FP32 direct-difference re-measure of the best candidate when the TF32
//     interval is not already decisive (u1 > 0.85 T or the rest within 2 u1);
//   * the row's in-batch distance columns to residuals at earlier positions
//     (<= RC_MAX residuals; more go to the tiled SIMT kernel), as k_res_cols.
// Each lane sums at most 4 NV <= 64 squared differences sequentially, then a
// 5-level warp tree: within the SIMT screen model screen_rel(D).
template <int NV, int MINB>
__global__ void __launch_bounds__(256, MINB) k_rowpass(int nA, int64_t a0, const char *const *__restrict__ frow, int D,
                                                const int64_t *__restrict__ ctr, const float *__restrict__ dist,
                                                int64_t ld, const float *__restrict__ cn2, const int32_t *__restrict__ snap,
                                                const float *__restrict__ fnorm, ScreenModel sm, float rel, float absc,
                                                const float *__restrict__ C32, double T, const int32_t *__restrict__ res_pos,
                                                float *__restrict__ dres, int64_t ldr, int32_t *__restrict__ sum_slot,
                                                int32_t *__restrict__ sum_q,
                                                float *__restrict__ sum_d1, float *__restrict__ sum_e1,
                                                float *__restrict__ sum_lbr, const float *__restrict__ snorm) {
    pdl_enter();
    __shared__ int s_rpos[RC_MAX];
    __shared__ int s_pmin;
    const int nsnap = (int)ctr[C_NSNAP];
    const int nres_all = (int)ctr[C_NRES];
    const int nres = nres_all <= RC_MAX ? nres_all : 0;  // more: the tiled kernel writes the columns
    if (threadIdx.x == 0) s_pmin = INT_MAX;
    __syncthreads();
    for (int r = threadIdx.x; r < nres; r += blockDim.x) {
        s_rpos[r] = res_pos[r];
        atomicMin(&s_pmin, res_pos[r]);
    }
    __syncthreads();
    const int pmin = s_pmin;
    const int lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    for (int w = blockIdx.x * nw + (threadIdx.x >> 5); w < nA; w += gridDim.x * nw) {
        const float fn = fnorm[a0 + w];
        // the row's features are needed whenever the TC screen ran (refine):
        // their loads fly while the distance row is scanned
        const float4 *f4 = (const float4 *)frow[a0 + w];
        float4 x[NV];
        const bool pre = sm.tc && nsnap > 0;
        if (pre) {
#pragma unroll
            for (int j = 0; j < NV; j++) {
                const int e = lane + 32 * j;
                x[j] = (4 * e < D) ? __ldg(f4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float u1, l1, lbr;
        int q1;
        row_scan(dist + (int64_t)w * ld, nsnap, cn2, snap, snorm, sm, fn, lane, u1, l1, lbr, q1);
        float d1 = 0.5f * (l1 + u1), e1 = 0.5f * (u1 - l1);
        const bool refine = sm.tc && q1 >= 0;  // a tight ub0 keeps the resolve's drift bounds small
        const bool cols = nres > 0 && w > pmin;
        if (refine || cols) {
            if (!pre) {
#pragma unroll
                for (int j = 0; j < NV; j++) {
                    const int e = lane + 32 * j;
                    x[j] = (4 * e < D) ? __ldg(f4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            auto dist_to = [&](const float4 *c4) {
                float acc = 0.f;
#pragma unroll
                for (int j = 0; j < NV; j++) {
                    const int e = lane + 32 * j;
                    if (4 * e < D) {
                        const float4 c = __ldg(c4 + e);
                        float d = x[j].x - c.x;
                        acc = fmaf(d, d, acc);
                        d = x[j].y - c.y;
                        acc = fmaf(d, d, acc);
                        d = x[j].z - c.z;
                        acc = fmaf(d, d, acc);
                        d = x[j].w - c.w;
                        acc = fmaf(d, d, acc);
                    }
                }
                return sqrtf(warp_sum(acc));
            };
            if (refine) {
                const float dd = dist_to((const float4 *)(C32 + (int64_t)snap[q1] * D));
                const float ee = rel * dd + absc * (sqrtf(cn2[snap[q1]]) * 1.00001f + fn) + 1e-30f;
                if (dd + ee < u1) {  // keep whichever interval is tighter (both are valid)
                    d1 = dd;
                    e1 = ee;
                }
            }
            if (cols) {
                for (int r = 0; r < nres; r++) {
                    const int rp = s_rpos[r];
                    if (rp >= w) continue;
                    const float v = dist_to((const float4 *)frow[a0 + rp]);
                    if (lane == 0) dres[(int64_t)w * ldr + r] = v;
                }
            }
        }
        if (lane == 0) {
            sum_slot[w] = q1 >= 0 ? snap[q1] : -1;
            sum_q[w] = q1;
            sum_d1[w] = d1;
            sum_e1[w] = e1;
            sum_lbr[w] = lbr;
        }
    }
}

// Lean row pass (D <= 2048, fp32 rows, 16-byte aligned): the same outputs as
// k_rowpass<16> with the same arithmetic order (each lane's 64 squared
// differences summed sequentially, then the warp tree), but the row is not
// held in registers across the distance-row scan: it is streamed in quarters
// together with the centroid row, so the kernel fits 4 CTAs per SM (one
// wave for a batch of 8192) instead of 2.
__global__ void __launch_bounds__(256, 4) k_rowpass_lean(int nA, int64_t a0, const char *const *__restrict__ frow,
                                                        int D, const int64_t *__restrict__ ctr,
                                                        const float *__restrict__ dist, int64_t ld,
                                                        const float *__restrict__ cn2, const int32_t *__restrict__ snap,
                                                        const float *__restrict__ fnorm, ScreenModel sm, float rel,
                                                        float absc, const float *__restrict__ C32, double T,
                                                        const int32_t *__restrict__ res_pos, float *__restrict__ dres,
                                                        int64_t ldr, int32_t *__restrict__ sum_slot,
                                                        int32_t *__restrict__ sum_q, float *__restrict__ sum_d1,
                                                        float *__restrict__ sum_e1, float *__restrict__ sum_lbr,
                                                        const float *__restrict__ snorm) {
    pdl_enter();
    constexpr int NV = 16, QV = 4;  // float4 per lane per row, per quarter
    __shared__ int s_rpos[RC_MAX];
    __shared__ int s_pmin;
    const int nsnap = (int)ctr[C_NSNAP];
    const int nres_all = (int)ctr[C_NRES];
    const int nres = nres_all <= RC_MAX ? nres_all : 0;  // more: the tiled kernel writes the columns
    if (threadIdx.x == 0) s_pmin = INT_MAX;
    __syncthreads();
    for (int r = threadIdx.x; r < nres; r += blockDim.x) {
        s_rpos[r] = res_pos[r];
        atomicMin(&s_pmin, res_pos[r]);
    }
    __syncthreads();
    const int pmin = s_pmin;
    const int lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    for (int w = blockIdx.x * nw + (threadIdx.x >> 5); w < nA; w += gridDim.x * nw) {
        const float fn = fnorm[a0 + w];
        const float4 *f4 = (const float4 *)frow[a0 + w];
        float u1, l1, lbr;
        int q1;
        row_scan(dist + (int64_t)w * ld, nsnap, cn2, snap, snorm, sm, fn, lane, u1, l1, lbr, q1);
        float d1 = 0.5f * (l1 + u1), e1 = 0.5f * (u1 - l1);
        auto dist_to = [&](const float4 *c4) {
            float acc = 0.f;
#pragma unroll 1
            for (int j0 = 0; j0 < NV; j0 += QV) {
                float4 x[QV], c[QV];
#pragma unroll
                for (int j = 0; j < QV; j++) {
                    const int e = lane + 32 * (j0 + j);
                    const bool in = 4 * e < D;
                    x[j] = in ? __ldg(f4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                    c[j] = in ? __ldg(c4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int j = 0; j < QV; j++) {
                    if (4 * (lane + 32 * (j0 + j)) < D) {
                        float d = x[j].x - c[j].x;
                        acc = fmaf(d, d, acc);
                        d = x[j].y - c[j].y;
                        acc = fmaf(d, d, acc);
                        d = x[j].z - c[j].z;
                        acc = fmaf(d, d, acc);
                        d = x[j].w - c[j].w;
                        acc = fmaf(d, d, acc);
                    }
                }
            }
            return sqrtf(warp_sum(acc));
        };
        if (sm.tc && q1 >= 0) {  // a tight ub0 keeps the resolve's drift bounds small
            const float dd = dist_to((const float4 *)(C32 + (int64_t)snap[q1] * D));
            const float ee = rel * dd + absc * (sqrtf(cn2[snap[q1]]) * 1.00001f + fn) + 1e-30f;
            if (dd + ee < u1) {  // keep whichever interval is tighter (both are valid)
                d1 = dd;
                e1 = ee;
            }
        }
        if (nres > 0 && w > pmin) {
            for (int r = 0; r < nres; r++) {
                const int rp = s_rpos[r];
                if (rp >= w) continue;
                const float v = dist_to((const float4 *)frow[a0 + rp]);
                if (lane == 0) dres[(int64_t)w * ldr + r] = v;
            }
        }
        if (lane == 0) {
            sum_slot[w] = q1 >= 0 ? snap[q1] : -1;
            sum_q[w] = q1;
            sum_d1[w] = d1;
            sum_e1[w] = e1;
            sum_lbr[w] = lbr;
        }
    }
}

// Wide row pass for large snapshots (C3: 100 k live centroids): one CTA per
// object, the distance row split over 8 warps (row_scan per segment, merged
// in warp order with row_scan's tie rule), then warp 0 refines the best
// candidate exactly as k_rowpass_lean.  Residual columns are left to the
// tiled kernel (this variant runs only when there are none to do here).
constexpr int RPW_T = 256, RPW_W = RPW_T / 32;
__global__ void __launch_bounds__(RPW_T) k_rowpass_wide(int nA, int64_t a0, const char *const *__restrict__ frow,
                                                       int D, const int64_t *__restrict__ ctr,
                                                       const float *__restrict__ dist, int64_t ld,
                                                       const float *__restrict__ cn2, const int32_t *__restrict__ snap,
                                                       const float *__restrict__ fnorm, ScreenModel sm, float rel,
                                                       float absc, const float *__restrict__ C32,
                                                       int32_t *__restrict__ sum_slot, int32_t *__restrict__ sum_q,
                                                       float *__restrict__ sum_d1, float *__restrict__ sum_e1,
                                                       float *__restrict__ sum_lbr, const float *__restrict__ snorm) {
    pdl_enter();
    __shared__ float s_u[RPW_W], s_l[RPW_W], s_r[RPW_W];
    __shared__ int s_q[RPW_W];
    const int nsnap = (int)ctr[C_NSNAP];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int w = blockIdx.x; w < nA; w += gridDim.x) {
        const float fn = fnorm[a0 + w];
        const int seg = ((nsnap + RPW_W - 1) / RPW_W + 255) & ~255;  // whole 32 x 8 row_scan steps
        const int qb = wid * seg, qe = min(nsnap, qb + seg);
        float u1, l1, lbr;
        int q1;
        row_scan(dist + (int64_t)w * ld, qe, cn2, snap, snorm, sm, fn, lane, u1, l1, lbr, q1, qb);
        if (lane == 0) {
            s_u[wid] = u1;
            s_l[wid] = l1;
            s_r[wid] = lbr;
            s_q[wid] = q1;
        }
        __syncthreads();
        if (wid == 0) {
            u1 = s_u[0];
            l1 = s_l[0];
            lbr = s_r[0];
            q1 = s_q[0];
            for (int v = 1; v < RPW_W; v++) {
                const float ou = s_u[v], ol = s_l[v], olbr = s_r[v];
                const int oq = s_q[v];
                const bool take = oq >= 0 && (q1 < 0 || ou < u1 || (ou == u1 && oq < q1));
                if (take) {
                    lbr = fminf(fminf(lbr, olbr), q1 >= 0 ? l1 : INFINITY);
                    u1 = ou;
                    l1 = ol;
                    q1 = oq;
                } else {
                    lbr = fminf(fminf(lbr, olbr), oq >= 0 ? ol : INFINITY);
                }
            }
            float d1 = 0.5f * (l1 + u1), e1 = 0.5f * (u1 - l1);
            if (sm.tc && q1 >= 0) {
                const float4 *f4 = (const float4 *)frow[a0 + w];
                const float4 *c4 = (const float4 *)(C32 + (int64_t)snap[q1] * D);
                float acc = 0.f;
#pragma unroll 1
                for (int j0 = 0; j0 < 16; j0 += 4) {
                    float4 x[4], c[4];
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const int e = lane + 32 * (j0 + j);
                        const bool in = 4 * e < D;
                        x[j] = in ? __ldg(f4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                        c[j] = in ? __ldg(c4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        if (4 * (lane + 32 * (j0 + j)) < D) {
                            float d = x[j].x - c[j].x;
                            acc = fmaf(d, d, acc);
                            d = x[j].y - c[j].y;
                            acc = fmaf(d, d, acc);
                            d = x[j].z - c[j].z;
                            acc = fmaf(d, d, acc);
                            d = x[j].w - c[j].w;
                            acc = fmaf(d, d, acc);
                        }
                    }
                }
                const float dd = sqrtf(warp_sum(acc));
                const float ee = rel * dd + absc * (sqrtf(cn2[snap[q1]]) * 1.00001f + fn) + 1e-30f;
                if (dd + ee < u1) {
                    d1 = dd;
                    e1 = ee;
                }
            }
            if (lane == 0) {
                sum_slot[w] = q1 >= 0 ? snap[q1] : -1;
                sum_q[w] = q1;
                sum_d1[w] = d1;
                sum_e1[w] = e1;
                sum_lbr[w] = lbr;
            }
        }
        __syncthreads();
    }
}

constexpr int RS_MAXGRP = 512;
constexpr int RS_RANKW = 8;
#ifndef RS_UB_SCAN
#define RS_UB_SCAN 1  // 0: i*U instead of per-object prefix sums of hypothesis bounds (tighter drift, one more scan)
#endif  // warps that rank a window (per-warp group counters)
constexpr int RS_WCNT_BYTES = RS_RANKW * RS_MAXGRP * 2;
constexpr int RS_WIN0 = 64;

// Drift bound for a group inside one window.  With c_ref the point the
// hypothesis bounds refer to (snapshot centroid, or the seed's feature) and
// c_w the slot's centroid at window start (|c_w - c_ref| <= d0, nf0 featured
// members), after i more joins the centroid is the exact mean
//   c_i = (nf0 c_w + sum_{q<i} f_q) / (nf0 + i),
// so |c_i - c_ref| <= (nf0 d0 + sum_{q<i} |f_q - c_ref|) / (nf0 + i) and
// |f_q - c_ref| <= ub0_q (P = that sum of bounds).  The float64 rounding of
// the i running-sum adds and of the two divisions adds at most
// (i + 4) 4u (2|c| + d0 + U) (u = 2^-53, U = largest ub0 of the group).
__device__ __forceinline__ float drift_avg(float d0, int nf0, float P, int i, float cn, float U) {
    const double n = (double)nf0 + (double)i;
    const double core = ((double)nf0 * (double)d0 + (double)P) / n;
    const double slack = ((double)i + 4.0) * 4.0 * 1.1102230246251565e-16 * (2.0 * (double)cn + (double)d0 + (double)U);
    return __double2float_ru((core + slack) * (1.0 + 1e-12));
}

// Segmented exclusive scan (fp32, every add rounded up -> an upper bound of
// the exact sum) of val[list[j]] over list positions j in [0, n); a segment
// starts where the group id changes.  Whole block; out[j] by list position.
__device__ void seg_scan_ub(int n, const int32_t *list, const short *grp, const float *val, float *out, float *wsf,
                            int *wsh) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nthr = blockDim.x;
    const int per = (n + nthr - 1) / nthr;
    const int jlo = min(n, tid * per), jhi = min(n, jlo + per);
    float run = 0.f;
    int head = 0;
    for (int j = jlo; j < jhi; j++) {
        const int p = list[j];
        if (j == 0 || grp[list[j - 1]] != grp[p]) {
            run = 0.f;
            head = 1;
        }
        out[j] = run;
        run = __fadd_ru(run, val[p]);
    }
    float v = run;
    int h = head;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float vp = __shfl_up_sync(0xffffffffu, v, o);
        const int hp = __shfl_up_sync(0xffffffffu, h, o);
        if (lane >= o) {
            if (!h) v = __fadd_ru(v, vp);
            h |= hp;
        }
    }
    if (lane == 31) {
        wsf[wid] = v;
        wsh[wid] = h;
    }
    float ve = __shfl_up_sync(0xffffffffu, v, 1);
    int he = __shfl_up_sync(0xffffffffu, h, 1);
    if (lane == 0) {
        ve = 0.f;
        he = 0;
    }
    __syncthreads();
    if (tid == 0) {
        float cv = 0.f;
        int ch = 0;
        for (int w = 0; w < (nthr >> 5); w++) {
            const float tv = wsf[w];
            const int th = wsh[w];
            wsf[w] = cv;
            wsh[w] = ch;
            cv = th ? tv : __fadd_ru(cv, tv);
            ch |= th;
        }
    }
    __syncthreads();
    const float carry = he ? ve : __fadd_ru(wsf[wid], ve);
    for (int j = jlo; j < jhi; j++) {
        if (j == 0 || grp[list[j - 1]] != grp[list[j]]) break;
        out[j] = __fadd_ru(out[j], carry);
    }
    __syncthreads();
}

__device__ __forceinline__ double drift_step(double dr, double ub, int nf, double cn) {
    // ||c_new - c_old|| <= ub / nf in exact arithmetic (c' - c = (f - c)/n');
    // 8 u64 (|c| + dr + ub) covers the float64 rounding of the sum and of S/n.
    return dr + ub / nf + 8.0 * 1.1102230246251565e-16 * (cn + dr + ub) + 1e-300;
}

// Ordered block compaction of [lo, hi) (hi - lo <= 4096): out[r] = the r-th i
// with pred(i).  Returns the count (every thread).
template <class Pred>
__device__ int rs_compact(int lo, int hi, Pred pred, int32_t *out, int *wsv, int *s_tot) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (hi - lo + RS_THREADS - 1) / RS_THREADS;
    const int i0 = min(hi, lo + tid * per), i1 = min(hi, i0 + per);
    int c = 0;
    for (int i = i0; i < i1; i++) c += pred(i) ? 1 : 0;
    int v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) wsv[wid] = v;
    __syncthreads();
    if (tid == 0) {
        int a = 0;
        for (int w = 0; w < RS_WARPS; w++) {
            const int t = wsv[w];
            wsv[w] = a;
            a += t;
        }
        *s_tot = a;
    }
    __syncthreads();
    int r = wsv[wid] + v - c;
    for (int i = i0; i < i1; i++)
        if (pred(i)) out[r++] = i;
    const int tot = *s_tot;
    __syncthreads();
    return tot;
}

template <typename T>
__global__ void __launch_bounds__(RS_THREADS, 1) k_resolve(ResolveArgs A) {
    pdl_enter();
    {  // the fast path (k_rfast1/k_rfast3) committed this batch: nothing to do
        const int64_t fst = A.ctr[C_FASTST];
        __syncthreads();
        if (threadIdx.x == 0) A.ctr[C_FASTST] = 0;
        if (fst == 1) return;
    }
    // the exact path reads and writes the reference's float64 sums S: the
    // previous batch's lagged chain (k_fold, second stream) must be done.
    // Waiting here instead of on the stream keeps the fast path off the
    // chain (the chain needs no SM this CTA holds, so it always progresses).
    if (A.chain_epoch) {
        if (threadIdx.x == 0) {
            while (*(volatile const unsigned long long *)A.chain_epoch < (unsigned long long)A.batch_no)
                __nanosleep(200);
            __threadfence();
        }
        __syncthreads();
    }

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int B = A.B;
    const int BC = A.Bcap;  // layout by capacity (multiple of 64): every array stays aligned
    unsigned short *wcnt = (unsigned short *)smem_raw;    // [RS_RANKW][RS_MAXGRP] per-warp group counts
    // per-object state: shared memory up to 4096 objects, else global (A.rs_gobj)
    unsigned char *obj_base = A.rs_gobj ? A.rs_gobj : smem_raw + RS_WCNT_BYTES;
    int32_t *sh_slot_of = (int32_t *)obj_base;             // [B]
    int *mlist = (int *)(sh_slot_of + BC);                 // [B]
    int32_t *seg_key = (int32_t *)(mlist + BC);            // [B] hypothesis slot
    float *seg_ub0 = (float *)(seg_key + BC);              // [B] d1 + e1
    float *seg_lbr = (float *)(seg_ub0 + BC);              // [B] min over others of d - e
    int32_t *seedlist = (int32_t *)(seg_lbr + BC);         // [B] in-batch seed slots
    int32_t *seg_nf = seedlist + BC;                       // [B] rank inside the hypothesis group
    int32_t *glist = seg_nf + BC;                         // [B] group-ordered positions
    float *seg_P = (float *)(glist + BC);                 // [B] by list position: sum of ub0 over earlier group members
    short *seg_grp = (short *)(seg_P + BC);               // [B]
    unsigned char *seg_flag = (unsigned char *)(seg_grp + BC);  // [B]
    double *scratch = (double *)(seg_flag + BC);          // pairwise scratch
    __shared__ Cand red[RS_WARPS];
    __shared__ int cand_list[RS_MAXCAND];
    __shared__ int n_cand;
    __shared__ int s_L, s_nfree, s_ndefer, s_nevict, s_nod, s_ndirty, s_nseeds, s_any_evicted;
    __shared__ long long s_dc, s_exact, s_fast, s_next_cid, s_inserted, s_victim_key;
    __shared__ int s_decision_slot, s_seed, s_need_exact, s_need_evict, s_need_od;
    __shared__ double s_best_d;
    __shared__ int s_best_slot;
    __shared__ float s_ub_used;
    __shared__ int grp_slot[RS_MAXGRP];
    __shared__ int grp_cnt[RS_MAXGRP], grp_off[RS_MAXGRP], grp_ncommit[RS_MAXGRP], grp_nf0[RS_MAXGRP];
    __shared__ int grp_cid[RS_MAXGRP], grp_size0[RS_MAXGRP], grp_pend0[RS_MAXGRP];
    __shared__ float grp_drift[RS_MAXGRP], grp_U[RS_MAXGRP], grp_d0[RS_MAXGRP], grp_cn[RS_MAXGRP];
    __shared__ int s_ngrp, s_fail, s_tot, s_nold, s_conf, s_scan, s_cfirst;
    __shared__ unsigned s_zmask[128];  // window seeds without dedup followers (bit k)
    __shared__ double s_md1, s_md2;
    __shared__ int s_md1_slot;
    __shared__ double wmd1[RS_WARPS], wmd2[RS_WARPS];
    __shared__ int wmds[RS_WARPS], wsv[RS_WARPS], wsh[RS_WARPS];
    __shared__ float wsf[RS_WARPS];

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int64_t *ctr = A.ctr;

    // ---- batch prologue: recycle last batch's freed slots, reset snapshot fields
    if (tid == 0) {
        s_L = (int)ctr[C_NLIVE];
        s_nfree = (int)ctr[C_NFREE];
        int nd = (int)ctr[C_NDEFER];
        for (int i = 0; i < nd; i++) A.free_stack[s_nfree++] = A.defer_free[i];
        s_ndefer = 0;
        s_nevict = 0;
        s_nod = 0;
        s_ndirty = 0;
        s_nseeds = 0;
        s_any_evicted = 0;
        s_dc = ctr[C_DC];
        s_exact = ctr[C_EXACT];
        s_fast = ctr[C_FAST];
        s_next_cid = ctr[C_NEXT_CID];
        s_inserted = ctr[C_NINSERTED];
    }
    __syncthreads();
    const int nsnap = (int)ctr[C_NSNAP];
    for (int q = tid; q < nsnap; q += blockDim.x) {
        int sl = A.snap_slot[q];
        A.s_snapq[sl] = q;
        A.s_seedpos[sl] = -1;
        A.s_foldpos[sl] = 0;
        A.s_pend[sl] = 0;
        A.s_odcol[sl] = -1;
        A.s_drift[sl] = A.s_sdev[sl];  // the snapshot's distance from the exact centroid (k_tfold)
    }
    for (int b = tid; b < B; b += blockDim.x) sh_slot_of[b] = -1;
    __syncthreads();

    int b = 0, win = min(B, 4096);  // first window: the whole batch up to 4096 (failures shrink it)
    while (b < B) {
        // =================== parallel segment: speculate every object in
        // [b, e_end) joins its nearest candidate, verify with bounds, commit
        // the verified prefix ===================
        const int e_end = min(B, b + win);
        const int L = s_L;
        long long t0 = clock64();
        if (tid == 0) {
            s_ngrp = 0;
            s_fail = e_end;
            A.prof[6]++;
        }
        // pass A: hypothesis per object (snapshot summary + in-batch seeds).
        // With no in-batch seed and no eviction yet every hypothesis is a
        // snapshot slot: its snapshot index is the group id (no slot map).
        const bool qkeys = s_nseeds == 0 && !s_any_evicted && nsnap <= RS_MAXGRP;
        if (s_nseeds == 0 && !s_any_evicted) {
#pragma unroll 4
            for (int p = b + tid; p < e_end; p += blockDim.x) {
                const float d1 = A.sum_d1[p], e1 = A.sum_e1[p], lbr = A.sum_lbr[p];
                seg_key[p] = (L > 0) ? A.sum_slot[p] : -1;
                if (qkeys) seg_grp[p] = (short)((L > 0) ? A.sum_q[p] : -1);
                seg_ub0[p] = (d1 + e1) * 1.000001f + 1e-30f;
                seg_lbr[p] = lbr - fabsf(lbr) * 1e-6f - 1e-30f;
                const float lball = (L > 0) ? fminf(d1 - e1, lbr) : INFINITY;
                if (A.res_col[p] >= 0 && (double)lball > A.T) {
                    // probable seed: no candidate can join it; kept out of the groups
                    seg_key[p] = -1;
                    if (qkeys) seg_grp[p] = -1;
                    seg_lbr[p] = lball - fabsf(lball) * 1e-6f - 1e-30f;
                }
            }
        } else
        for (int p = b + tid; p < e_end; p += blockDim.x) {
            const float fn = A.fnorm[A.c0 + p];
            int j1 = A.sum_slot[p];
            float d1 = A.sum_d1[p], e1 = A.sum_e1[p], lbr = A.sum_lbr[p];
            if (s_any_evicted && j1 >= 0 && A.s_evicted[j1] && A.res_col[p] >= 0) {
                // probable-seed pre-test before any rescan: the snapshot summary
                // bounds a superset of the live clusters
                float lb = fminf(d1 - e1, lbr);
                for (int k = 0; k < s_nseeds && (double)lb > A.T; k++) {
                    const int sl = seedlist[k];
                    if (A.s_evicted[sl]) continue;
                    const int s = A.s_seedpos[sl];
                    const int col = A.res_col[s];
                    const float d = col >= 0 ? A.dres[(int64_t)p * A.ldr + col] : A.dod[(int64_t)A.s_odcol[sl] * B + p];
                    lb = fminf(lb, d - (A.rel * d + A.absc * (A.fnorm[A.c0 + s] + fn) + 1e-30f));
                }
                if ((double)lb > A.T) {
                    seg_key[p] = -1;
                    seg_ub0[p] = INFINITY;
                    seg_lbr[p] = lb - fabsf(lb) * 1e-6f - 1e-30f;
                    continue;
                }
            }
            if (s_any_evicted && (j1 < 0 || A.s_evicted[j1])) {
                j1 = -1;
                d1 = INFINITY;
                lbr = INFINITY;
                for (int i = 0; i < L; i++) {
                    const int sl = A.live[i];
                    const int q = A.s_snapq[sl];
                    if (q < 0) continue;
                    float l0, u0;
                    snap_bounds(A.sm, A.dist[(int64_t)p * A.ld + q], sqrtf(A.s_cn2[sl]) * 1.00001f, fn, l0, u0);
                    const float d = 0.5f * (l0 + u0), e = 0.5f * (u0 - l0);
                    if (u0 < d1 + e1 || j1 < 0) {
                        if (j1 >= 0) lbr = fminf(lbr, d1 - e1);
                        j1 = sl;
                        d1 = d;
                        e1 = e;
                    } else {
                        lbr = fminf(lbr, l0);
                    }
                }
            }
            for (int k = 0; k < s_nseeds; k++) {
                const int sl = seedlist[k];
                if (A.s_evicted[sl]) continue;
                const int s = A.s_seedpos[sl];
                const int col = A.res_col[s];
                const float d = col >= 0 ? A.dres[(int64_t)p * A.ldr + col] : A.dod[(int64_t)A.s_odcol[sl] * B + p];
                const float e = A.rel * d + A.absc * (A.fnorm[A.c0 + s] + fn) + 1e-30f;
                if (d < d1) {
                    if (j1 >= 0) lbr = fminf(lbr, d1 - e1);
                    j1 = sl;
                    d1 = d;
                    e1 = e;
                } else {
                    lbr = fminf(lbr, d - e);
                }
            }
            seg_key[p] = (L > 0) ? j1 : -1;
            seg_ub0[p] = (d1 + e1) * 1.000001f + 1e-30f;
            seg_lbr[p] = lbr - fabsf(lbr) * 1e-6f - 1e-30f;
            const float lball = (L > 0) ? fminf(d1 - e1, lbr) : INFINITY;
            if (A.res_col[p] >= 0 && (double)lball > A.T) {  // probable seed (see above)
                seg_key[p] = -1;
                seg_lbr[p] = lball - fabsf(lball) * 1e-6f - 1e-30f;
            }
        }
        for (int g = tid; g < RS_MAXGRP; g += blockDim.x) {
            grp_cnt[g] = 0;
            grp_U[g] = 0.f;
        }
        __syncthreads();
        long long t1 = clock64();
        if (tid == 0) A.prof[0] += t1 - t0;
        // pass B1: distinct hypothesis slots -> group ids; per group the
        // largest hypothesis upper bound (it bounds every member's join step)
        if (qkeys) {
            if (tid == 0) s_ngrp = nsnap;
            for (int g = tid; g < nsnap; g += blockDim.x) grp_slot[g] = A.snap_slot[g];
        } else {
            for (int p = b + tid; p < e_end; p += blockDim.x) {
                const int key = seg_key[p];
                if (key < 0) continue;
                if (A.s_grp[key] == -1 && atomicCAS(&A.s_grp[key], -1, -2) == -1) {
                    int g = atomicAdd(&s_ngrp, 1);
                    if (g < RS_MAXGRP) grp_slot[g] = key;
                    A.s_grp[key] = g < RS_MAXGRP ? g : RS_MAXGRP;
                }
            }
        }
        __syncthreads();
        const int ngrp = min(s_ngrp, RS_MAXGRP);
        const bool overflow = s_ngrp > RS_MAXGRP;
        for (int p = b + tid; p < e_end; p += blockDim.x) {
            int g;
            if (qkeys) {
                g = seg_grp[p];
            } else {
                const int key = seg_key[p];
                g = key >= 0 ? A.s_grp[key] : -1;
                g = (g >= 0 && g < RS_MAXGRP) ? g : -1;
                seg_grp[p] = (short)g;
            }
            if (g >= 0) atomicMax((int *)&grp_U[g], __float_as_int(seg_ub0[p]));  // ub0 > 0
        }
        for (int g = tid; g < ngrp; g += blockDim.x) {
            const int sl = grp_slot[g];
            grp_nf0[g] = A.s_nfeat[sl];
            grp_d0[g] = __double2float_ru(A.s_drift[sl]);
            grp_cn[g] = sqrtf(A.s_cn2[sl]) * 1.00001f;
            grp_cid[g] = A.s_cid[sl];
            grp_size0[g] = A.s_size[sl];
            grp_pend0[g] = A.s_pend[sl];
        }
        __syncthreads();
        // pass B2: stable rank of every object inside its group.  Each warp
        // ranks a contiguous chunk (match per 32-slice, warp-private counts),
        // an exclusive scan over warps per group gives the chunk bases.
        const int nwin = e_end - b;
        const int cs = ((nwin + RS_RANKW * 32 - 1) / (RS_RANKW * 32)) * 32;
        if (!overflow) {
            for (int e = tid; e < RS_RANKW * ngrp; e += blockDim.x) wcnt[e] = 0;
            __syncthreads();
            const int lo = wid < RS_RANKW ? b + wid * cs : e_end, hi = min(e_end, lo + cs);
            for (int p0 = lo; p0 < hi; p0 += 32) {
                const int p = p0 + lane;
                const int g = p < hi ? seg_grp[p] : -1;
                const unsigned act = __ballot_sync(0xffffffffu, g >= 0);
                unsigned lower = 0, peers = 0;
                if (g >= 0) {
                    peers = __match_any_sync(act, g);
                    lower = peers & ((1u << lane) - 1u);
                    seg_nf[p] = wcnt[wid * ngrp + g] + __popc(lower);
                }
                __syncwarp();
                if (g >= 0 && lower == 0) wcnt[wid * ngrp + g] += (unsigned short)__popc(peers);
                __syncwarp();
            }
            __syncthreads();
            for (int g = tid; g < ngrp; g += blockDim.x) {
                int run = 0;
                for (int w = 0; w < RS_RANKW; w++) {
                    const int c = wcnt[w * ngrp + g];
                    wcnt[w * ngrp + g] = (unsigned short)run;
                    run += c;
                }
                grp_cnt[g] = run;
            }
            __syncthreads();
            for (int p = b + tid; p < e_end; p += blockDim.x) {
                const int g = seg_grp[p];
                if (g >= 0) seg_nf[p] += wcnt[((p - b) / cs) * ngrp + g];
            }
            if (wid == 0) {  // exclusive prefix over groups
                int run = 0;
                for (int g0 = 0; g0 < ngrp; g0 += 32) {
                    const int g = g0 + lane;
                    const int c = g < ngrp ? grp_cnt[g] : 0;
                    int x = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    if (g < ngrp) grp_off[g] = run + x - c;
                    run += __shfl_sync(0xffffffffu, x, 31);
                }
            }
            __syncthreads();
            for (int p = b + tid; p < e_end; p += blockDim.x) {
                const int g = seg_grp[p];
                if (g >= 0) glist[grp_off[g] + seg_nf[p]] = p;
            }
            __syncthreads();
            // per object: sum of the hypothesis bounds of the group's earlier
            // members (segmented exclusive scan over glist, fp32 rounded up)
            const int nlist = ngrp ? grp_off[ngrp - 1] + grp_cnt[ngrp - 1] : 0;
            if (RS_UB_SCAN) seg_scan_ub(nlist, glist, seg_grp, seg_ub0, seg_P, wsf, wsh);
            for (int g = tid; g < ngrp; g += blockDim.x) {
                const int jl = grp_off[g] + grp_cnt[g] - 1;
                const float Ptot = !RS_UB_SCAN ? __fmul_ru((float)grp_cnt[g], grp_U[g])
                                   : grp_cnt[g] > 0 ? __fadd_ru(seg_P[jl], seg_ub0[glist[jl]]) : 0.f;
                grp_drift[g] = drift_avg(grp_d0[g], grp_nf0[g], Ptot, grp_cnt[g], grp_cn[g], grp_U[g]);
            }
        }
        __syncthreads();
        long long t2 = clock64();
        if (tid == 0) A.prof[1] += t2 - t1;
        // pass C: the two largest end-of-segment drifts over live slots
        {
            double m1 = -1.0, m2 = -1.0;
            int m1s = -1;
            for (int i = tid; i < L; i += blockDim.x) {
                const int sl = A.live[i];
                const int g = qkeys ? A.s_snapq[sl] : A.s_grp[sl];
                const double d = (g >= 0 && g < RS_MAXGRP && g < ngrp && !overflow) ? (double)grp_drift[g] : A.s_drift[sl];
                if (d > m1) {
                    m2 = m1;
                    m1 = d;
                    m1s = sl;
                } else if (d > m2) {
                    m2 = d;
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double o1 = __shfl_xor_sync(0xffffffffu, m1, o), o2 = __shfl_xor_sync(0xffffffffu, m2, o);
                const int os = __shfl_xor_sync(0xffffffffu, m1s, o);
                if (o1 > m1) {
                    m2 = fmax(m1, o2);
                    m1 = o1;
                    m1s = os;
                } else {
                    m2 = fmax(m2, o1);
                }
            }
            if (lane == 0) {
                wmd1[wid] = m1;
                wmd2[wid] = m2;
                wmds[wid] = m1s;
            }
            __syncthreads();
            if (tid == 0) {
                double a1 = wmd1[0], a2 = wmd2[0];
                int as = wmds[0];
                for (int w = 1; w < RS_WARPS; w++) {
                    if (wmd1[w] > a1) {
                        a2 = fmax(a1, wmd2[w]);
                        a1 = wmd1[w];
                        as = wmds[w];
                    } else {
                        a2 = fmax(a2, wmd1[w]);
                    }
                }
                s_md1 = a1 < 0 ? 0.0 : a1;
                s_md2 = a2 < 0 ? 0.0 : a2;
                s_md1_slot = as;
            }
            __syncthreads();
        }
        // pass D: certainty check -> 0 certain, 1 only the T test is open
        // (confirmable by one exact distance), 2 anything else
        //         3 certain seed (no live centroid and no earlier probable seed of
        //         this window within T; evictions it causes are planned below).
        //         Probable seeds earlier in the window are candidates of every
        //         later object: their in-batch distance columns (dres) bound it.
        const int nres_w = (int)A.ctr[C_NRES];
        for (int p = b + tid; p < e_end; p += blockDim.x) {
            const int key = seg_key[p];
            unsigned char fl = 2;
            double ub = INFINITY;
            const bool seedc = key < 0 && A.res_col[p] >= 0 && !overflow;
            if (key >= 0 && !overflow) {
                const int g = seg_grp[p];
                const int i = seg_nf[p];
                const float Pi = RS_UB_SCAN ? seg_P[grp_off[g] + i] : __fmul_ru((float)i, grp_U[g]);
                ub = (double)seg_ub0[p] + (double)drift_avg(grp_d0[g], grp_nf0[g], Pi, i, grp_cn[g], grp_U[g]);
                const double md = (key == s_md1_slot) ? s_md2 : s_md1;
                const double lbo = (double)seg_lbr[p] - md * 1.000001;
                if (lbo > ub) fl = ub <= A.T ? 0 : 1;
            } else if (seedc) {
                if ((double)seg_lbr[p] - s_md1 * 1.000001 > A.T) fl = 3;
            }
            if (fl != 2 && nres_w > 0) {
                const float fnp = A.fnorm[A.c0 + p];
                for (int q = 0; q < nres_w; q++) {
                    const int pq = A.res_pos[q];
                    if (pq < b || pq >= p) continue;
                    if (A.res_col[pq] < 0 || seg_key[pq] >= 0) continue;  // not a probable seed of this window
                    const float d = A.dres[(int64_t)p * A.ldr + q];
                    const float lb = d - (A.rel * d + A.absc * (fnp + A.fnorm[A.c0 + pq])) - 1e-30f;
                    const double bound = fl == 3 ? A.T : ub;
                    if (!((double)(lb - fabsf(lb) * 1e-6f) > bound)) {
                        fl = 2;
                        break;
                    }
                }
            }
            seg_flag[p] = fl;
            sh_slot_of[p] = key;  // tentative, for materialisation by the exact path
        }
        __syncthreads();
        long long t3 = clock64();
        if (tid == 0) A.prof[2] += t3 - t2;
        // confirm T-only failures in order with one exact distance each
        int f = b;
        while (true) {
            if (tid == 0) s_fail = e_end;
            __syncthreads();
            for (int p = f + tid; p < e_end; p += blockDim.x)
                if (seg_flag[p] == 1 || seg_flag[p] == 2) atomicMin(&s_fail, p);
            __syncthreads();
            f = s_fail;
            if (f >= e_end || seg_flag[f] != 1) break;
            const double dx =
                exact_dist<T>(A, f, seg_key[f], sh_slot_of, mlist, scratch, grp_nf0[seg_grp[f]] + seg_nf[f]);
            if (tid == 0) {
                s_exact++;
                // diagnostics: batch bucket (0,1-7,8-15,16-31,32-63,64-127,128+) and young slots (nfeat < 16)
                const int bn = A.batch_no;
                const int bk = bn == 0 ? 0 : bn < 8 ? 1 : bn < 16 ? 2 : bn < 32 ? 3 : bn < 64 ? 4 : bn < 128 ? 5 : 6;
                A.prof[8 + bk]++;
                if (grp_nf0[seg_grp[f]] + seg_nf[f] < 16) A.prof[15]++;
            }
            if (dx > A.T) break;  // nearest is beyond T: the object seeds (sequential path)
            f++;
            __syncthreads();
        }
        __syncthreads();
        // ---- evictions caused by the certain seeds of [b, f) (clustering.py:139-144).
        // The victim is the live cluster of minimum (size, first in live order =
        // cid); the new seed has size 1 at that moment, so every victim has size
        // 1: it is the head of the FIFO of live size-1 clusters in cid order.
        // That FIFO holds the size-1 clusters of earlier windows (scanned from
        // the persistent cursor ctr[C_EVCUR]; every cid below it is evicted or
        // larger) ahead of this window's seeds that keep size 1.  An earlier
        // cluster joined inside the window would leave the FIFO at its join:
        // the window is cut at the eviction that reaches it (sequential step).
        int ws = 0, k0 = 0, nev = 0, nold = 0;
        if (!overflow && nres_w > 0) {
            ws = rs_compact(b, f, [&](int p) { return seg_flag[p] == 3; }, A.ev_pos, wsv, &s_tot);
            k0 = (int)min((int64_t)ws, max((int64_t)0, A.M - (int64_t)L));  // seeds k >= k0 evict
            nev = ws - k0;
        }
        if (nev > 0) {
            const int f0 = f;
            for (int p = b + tid; p < f0; p += blockDim.x) {
                const int key = seg_key[p];
                if (key >= 0) atomicMin(&A.s_fjoin[key], p);
            }
            if (tid == 0) {
                s_nold = 0;
                s_conf = 0;
                s_scan = (int)ctr[C_EVCUR];
            }
            __syncthreads();
            const int cid_end = (int)s_next_cid;  // first cid of this window's seeds
            while (true) {
                const int base = s_scan, n0 = s_nold;
                if (n0 >= nev || s_conf || base >= cid_end) break;
                const int cid = base + tid;
                bool valid = false, conf = false;
                int slot = -1;
                if (cid < cid_end) {
                    slot = A.cid_slot[cid];
                    valid = A.s_cid[slot] == cid && !A.s_evicted[slot] && A.s_size[slot] == 1;
                    conf = valid && A.s_fjoin[slot] < f0;
                }
                if (tid == 0) s_cfirst = RS_THREADS;
                __syncthreads();
                if (conf) atomicMin(&s_cfirst, tid);
                __syncthreads();
                const bool take = valid && tid < s_cfirst;
                const unsigned m = __ballot_sync(0xffffffffu, take);
                if (lane == 0) wsv[wid] = __popc(m);
                __syncthreads();
                if (tid == 0) {
                    int a = 0;
                    for (int w = 0; w < RS_WARPS; w++) {
                        const int t = wsv[w];
                        wsv[w] = a;
                        a += t;
                    }
                    s_tot = a;
                }
                __syncthreads();
                const int r = n0 + wsv[wid] + __popc(m & ((1u << lane) - 1));
                if (take && r < nev) {
                    A.ev_vic[r] = slot;
                    if (r == nev - 1) s_scan = cid + 1;
                }
                __syncthreads();
                if (tid == 0) {
                    if (n0 + s_tot >= nev) {
                        s_nold = nev;
                    } else {
                        s_nold = n0 + s_tot;
                        if (s_cfirst < RS_THREADS) {
                            s_conf = 1;
                            s_scan = base + s_cfirst;
                        } else {
                            s_scan = min(base + RS_THREADS, cid_end);
                        }
                    }
                }
                __syncthreads();
            }
            nold = s_nold;
            if (s_conf) {  // cut at the eviction that would take the joined cluster
                f = A.ev_pos[k0 + nold];
                ws = k0 + nold;
                nev = nold;
            }
            if (tid == 0) ctr[C_EVCUR] = s_scan;
            for (int p = b + tid; p < f0; p += blockDim.x) {
                const int key = seg_key[p];
                if (key >= 0) A.s_fjoin[key] = 0x7fffffff;
            }
            if (nev > nold) {
                // pops past the earlier windows' FIFO: this window's seeds.  Seed
                // k pushes itself; an evicting seed pops the head (itself when the
                // queue was empty); a seed with dedup followers that is not popped
                // leaves (size > 1).  Queue length w -> max(w + a, c) per seed,
                // composed by a warp scan.
                for (int i = tid; i < 128; i += blockDim.x) s_zmask[i] = 0;
                __syncthreads();
                for (int k = tid; k < ws; k += blockDim.x)
                    if (A.dup_run[A.c0 + A.ev_pos[k]] == 0) atomicOr(&s_zmask[k >> 5], 1u << (k & 31));
                __syncthreads();
                if (wid == 0) {
                    int *entry = (int *)seg_lbr;  // free after pass D
                    constexpr int NEG = -(1 << 28);
                    const int kw = k0 + nold;
                    const int fr = s_nfree;
                    int w = 0, ne = 0, nr = 0;
                    for (int c = 0; c < ws; c += 32) {
                        const int k = c + lane;
                        const bool in = k < ws;
                        const int z = in ? (int)((s_zmask[k >> 5] >> (k & 31)) & 1u) : 0;
                        const bool wpop = in && k >= kw;
                        int a = wpop ? z - 1 : z, cc = wpop ? 0 : NEG;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int ap = __shfl_up_sync(0xffffffffu, a, o), cp = __shfl_up_sync(0xffffffffu, cc, o);
                            if (lane >= o) {
                                cc = max(cp + a, cc);
                                a = ap + a;
                            }
                        }
                        int ae = __shfl_up_sync(0xffffffffu, a, 1), ce = __shfl_up_sync(0xffffffffu, cc, 1);
                        if (lane == 0) {
                            ae = 0;
                            ce = NEG;
                        }
                        const int wb = max(w + ae, ce);  // queue length before seed k
                        const bool self = wpop && wb == 0;
                        const bool ent = in && z && !self;
                        const bool pop = wpop && !self;
                        const unsigned me = __ballot_sync(0xffffffffu, ent), mp = __ballot_sync(0xffffffffu, pop);
                        const unsigned lt = (1u << lane) - 1;
                        if (ent) entry[ne + __popc(me & lt)] = k;
                        __syncwarp();
                        if (wpop) {
                            const int kv = self ? k : entry[nr + __popc(mp & lt)];
                            A.ev_vic[k - k0] = A.free_stack[fr - 1 - kv];
                        }
                        w = max(w + __shfl_sync(0xffffffffu, a, 31), __shfl_sync(0xffffffffu, cc, 31));
                        ne += __popc(me);
                        nr += __popc(mp);
                        __syncwarp();
                    }
                }
            }
            __syncthreads();
        }
        for (int p = f + tid; p < e_end; p += blockDim.x) sh_slot_of[p] = -1;
        long long t4 = clock64();
        if (tid == 0) A.prof[3] += t4 - t3;
        // pass E: commit [b, f).  Members of a group before f form a prefix of
        // its stream-ordered list; member i of group g gets featured rank
        // nf0 + i, pending rank pend0 + i and member rank size0 + i + (dups
        // attached to the group's earlier members: segmented scan over glist).
        if (!overflow) {
            for (int g = tid; g < ngrp; g += blockDim.x) {
                const int off = grp_off[g], cnt = grp_cnt[g];
                int lo = 0, hi = cnt;  // first list index with p >= f
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (glist[off + mid] < f) lo = mid + 1; else hi = mid;
                }
                grp_ncommit[g] = lo;
            }
            const int nlist = ngrp ? grp_off[ngrp - 1] + grp_cnt[ngrp - 1] : 0;
            // segmented exclusive scan of dup_run over glist -> mlist[j]
            {
                const int per = (nlist + RS_THREADS - 1) / RS_THREADS;
                const int jlo = min(nlist, tid * per), jhi = min(nlist, jlo + per);
                int run = 0, head = 0;
                constexpr int PERMAX = (4096 + RS_THREADS - 1) / RS_THREADS;  // windows never exceed 4096 objects
                int dr[PERMAX];
                const int32_t *__restrict__ dup_run = A.dup_run + A.c0;
#pragma unroll
                for (int u = 0; u < PERMAX; u++) dr[u] = jlo + u < jhi ? dup_run[glist[jlo + u]] : 0;  // loads in flight together
#pragma unroll
                for (int u = 0; u < PERMAX; u++) {
                    const int j = jlo + u;
                    if (j >= jhi) break;
                    const int p = glist[j];
                    if (j == 0 || seg_grp[glist[j - 1]] != seg_grp[p]) {
                        run = 0;
                        head = 1;
                    }
                    mlist[j] = run;
                    run += dr[u];
                }
                int v = run, h = head;  // inclusive warp scan, segmented operator
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int vp = __shfl_up_sync(0xffffffffu, v, o), hp = __shfl_up_sync(0xffffffffu, h, o);
                    if (lane >= o) {
                        if (!h) v += vp;
                        h |= hp;
                    }
                }
                if (lane == 31) {
                    wsv[wid] = v;
                    wsh[wid] = h;
                }
                int ve = __shfl_up_sync(0xffffffffu, v, 1), he = __shfl_up_sync(0xffffffffu, h, 1);
                if (lane == 0) {
                    ve = 0;
                    he = 0;
                }
                __syncthreads();
                if (tid == 0) {  // exclusive scan over warps
                    int cv = 0, ch = 0;
                    for (int w = 0; w < RS_WARPS; w++) {
                        const int tv = wsv[w], th = wsh[w];
                        wsv[w] = cv;
                        wsh[w] = ch;
                        cv = th ? tv : cv + tv;
                        ch |= th;
                    }
                }
                __syncthreads();
                const int carry = he ? ve : wsv[wid] + ve;  // combine(warp prefix, lane prefix)
                for (int j = jlo; j < jhi; j++) {
                    if (j == 0 || seg_grp[glist[j - 1]] != seg_grp[glist[j]]) break;
                    mlist[j] += carry;
                }
            }
            __syncthreads();
            {
                // per-object writes; the object-index loads of 4 list entries are
                // issued together (restrict: the outputs never alias the inputs)
                const int64_t *__restrict__ cls_obj = A.cls_obj + A.c0;
                int32_t *__restrict__ cluster_of = A.cluster_of;
                int32_t *__restrict__ mrank = A.mrank;
                int32_t *__restrict__ frank = A.frank;
                int32_t *__restrict__ pend_rank = A.pend_rank;
                int32_t *__restrict__ slot_of = A.slot_of;
                for (int j0 = tid; j0 < nlist; j0 += 4 * RS_THREADS) {
                    int64_t obj[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int j = j0 + u * RS_THREADS;
                        obj[u] = j < nlist ? cls_obj[glist[j]] : 0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int j = j0 + u * RS_THREADS;
                        if (j >= nlist) break;
                        const int p = glist[j];
                        const int g = seg_grp[p];
                        const int i = j - grp_off[g];
                        if (i >= grp_ncommit[g]) continue;
                        const int sl = grp_slot[g];
                        cluster_of[obj[u]] = grp_cid[g];
                        mrank[obj[u]] = grp_size0[g] + i + mlist[j];
                        frank[obj[u]] = grp_nf0[g] + i;
                        pend_rank[p] = grp_pend0[g] + i;
                        slot_of[p] = sl;
                        sh_slot_of[p] = sl;
                    }
                }
            }
            __syncthreads();
            for (int g = tid; g < ngrp; g += blockDim.x) {
                const int n_c = grp_ncommit[g];
                const int sl = grp_slot[g];
                if (n_c > 0) {
                    const int jl = grp_off[g] + n_c - 1;
                    const int dups = mlist[jl] + A.dup_run[A.c0 + glist[jl]];
                    const int pend0 = A.s_pend[sl];
                    const float Pc = RS_UB_SCAN ? __fadd_ru(seg_P[jl], seg_ub0[glist[jl]]) : __fmul_ru((float)n_c, grp_U[g]);
                    A.s_drift[sl] = (double)drift_avg(grp_d0[g], grp_nf0[g], Pc, n_c, grp_cn[g], grp_U[g]);
                    A.s_nfeat[sl] = grp_nf0[g] + n_c;
                    A.s_size[sl] += n_c + dups;
                    A.s_pend[sl] = pend0 + n_c;
                    if (pend0 == 0) {
                        const int di = atomicAdd(&s_ndirty, 1);
                        A.s_didx[sl] = di;
                        A.dirty[di] = sl;
                    }
                }
                if (!qkeys) A.s_grp[sl] = -1;
            }
        }
        if (overflow) {
            __syncthreads();
            for (int g = tid; g < ngrp; g += blockDim.x) A.s_grp[grp_slot[g]] = -1;
            for (int p = b + tid; p < e_end; p += blockDim.x) {
                const int key = seg_key[p];
                if (key >= 0 && A.s_grp[key] == RS_MAXGRP) A.s_grp[key] = -1;
            }
        }
        // certain seeds of [b, f), in stream order: the k-th takes the next free
        // slot and cluster id (clustering.py:122-125); the planned victims are
        // evicted and the surviving seeds fill their live positions, then append
        if (ws > 0) {
            __syncthreads();
            for (int k = tid; k < ws; k += blockDim.x) {
                const int p = A.ev_pos[k];
                const int slot = A.free_stack[s_nfree - 1 - k];
                const int cid = (int)(s_next_cid + k);
                const int64_t cc = A.c0 + p;
                const int64_t obj = A.cls_obj[cc];
                A.s_cid[slot] = cid;
                A.s_nfeat[slot] = 1;
                A.s_size[slot] = 1 + A.dup_run[cc];  // dedup members following the seed join it
                A.s_drift[slot] = 0.0;
                A.s_cn2[slot] = A.fnorm[cc] * A.fnorm[cc];
                A.s_snapq[slot] = -1;
                A.s_seedpos[slot] = p;
                A.s_foldpos[slot] = p;
                A.s_pend[slot] = 1;
                A.s_evicted[slot] = 0;
                A.s_odcol[slot] = -1;
                A.s_grp[slot] = -1;
                A.cid_slot[cid] = slot;
                seedlist[s_nseeds + k] = slot;
                const int di = atomicAdd(&s_ndirty, 1);
                A.s_didx[slot] = di;
                A.dirty[di] = slot;
                A.pend_rank[p] = 0;
                A.slot_of[p] = slot;
                sh_slot_of[p] = slot;
                A.cluster_of[obj] = cid;
                A.mrank[obj] = 0;
                A.frank[obj] = 0;
                // later objects of the window see it while the live count grows
                if (k < k0) atomicAdd((unsigned long long *)&s_dc, (unsigned long long)(f - 1 - p));
            }
            __syncthreads();
            for (int i = tid; i < nev; i += blockDim.x) {
                const int v = A.ev_vic[i];
                A.s_evicted[v] = 1;
                A.evict_slot[s_nevict + i] = v;
                A.evict_cid[s_nevict + i] = A.s_cid[v];
                A.defer_free[s_ndefer + i] = v;
                if (A.s_pend[v] == 0) {  // untouched this batch but needs its final centroid
                    const int di = atomicAdd(&s_ndirty, 1);
                    A.s_didx[v] = di;
                    A.dirty[di] = v;
                }
            }
            __syncthreads();
            const int fr = s_nfree;
            const int nsv = rs_compact(0, ws, [&](int k) { return !A.s_evicted[A.free_stack[fr - 1 - k]]; }, A.ev_pos,
                                       wsv, &s_tot);
            for (int t = tid; t < nsv; t += blockDim.x) {
                const int slot = A.free_stack[fr - 1 - A.ev_pos[t]];
                const int pos = t < nold ? A.live_pos[A.ev_vic[t]] : L + (t - nold);
                A.live[pos] = slot;
                A.live_pos[slot] = pos;
            }
            __syncthreads();
            if (tid == 0) {
                s_L = L + nsv - nold;
                s_nseeds += ws;
                s_next_cid += ws;
                s_nfree -= ws;
                s_nevict += nev;
                s_ndefer += nev;
                if (nev > 0) s_any_evicted = 1;
            }
        }
        if (tid == 0) {
            const long long nok = f - b;
            s_dc += (long long)L * nok;
            s_fast += nok;
            s_inserted += nok;
        }
        __syncthreads();
        if (tid == 0) A.prof[4] += clock64() - t4;
        if (f >= e_end) {
            b = e_end;
            win = min(win * 2, min(B, 4096));
            continue;
        }
        long long t5 = clock64();
        win = max(RS_WIN0, win / 4);
        b = f;
        // =================== sequential exact step for object b ===================
        {
        const float fn = A.fnorm[A.c0 + b];
        const int L = s_L;
        // ---- candidate scan
        Cand c{INFINITY, 0x7fffffff, INFINITY, -1, INFINITY};
        for (int i = tid; i < L; i += blockDim.x) {
            int slot = A.live[i];
            float lb, ub, d;
            slot_bounds<T>(A, b, fn, slot, lb, ub, d);
            Cand o{ub, i, lb, i, INFINITY};
            cand_merge(c, o);
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            Cand o;
            o.ub = __shfl_xor_sync(0xffffffffu, c.ub, off);
            o.ubi = __shfl_xor_sync(0xffffffffu, c.ubi, off);
            o.lb1 = __shfl_xor_sync(0xffffffffu, c.lb1, off);
            o.lb1i = __shfl_xor_sync(0xffffffffu, c.lb1i, off);
            o.lb2 = __shfl_xor_sync(0xffffffffu, c.lb2, off);
            cand_merge(c, o);
        }
        if (lane == 0) red[wid] = c;
        __syncthreads();
        if (tid == 0) {
            Cand r = red[0];
            for (int w = 1; w < RS_WARPS; w++) cand_merge(r, red[w]);
            s_dc += L;
            s_need_exact = 0;
            s_need_evict = 0;
            s_need_od = -1;
            s_seed = 0;
            s_decision_slot = -1;
            if (L == 0 || (double)r.lb1 > A.T) {
                s_seed = 1;
                s_fast++;
            } else if (r.lb2 > r.ub) {
                // unique possible argmin
                int slot = A.live[r.ubi];
                if ((double)r.ub <= A.T) {
                    s_decision_slot = slot;
                    s_ub_used = r.ub;
                    s_fast++;
                } else {
                    s_need_exact = 1;
                    cand_list[0] = r.ubi;
                    n_cand = 1;
                }
            } else {
                s_need_exact = 2;
                n_cand = 0;
                s_ub_used = r.ub;
            }
        }
        __syncthreads();
        if (s_need_exact) {
            if (s_need_exact == 2) {
                const float U = s_ub_used;
                for (int i = tid; i < L; i += blockDim.x) {
                    int slot = A.live[i];
                    float lb, ub, d;
                    slot_bounds<T>(A, b, fn, slot, lb, ub, d);
                    if (lb <= U) {
                        int p = atomicAdd(&n_cand, 1);
                        if (p < RS_MAXCAND) cand_list[p] = i;
                    }
                }
                __syncthreads();
            }
            const int nc = n_cand < RS_MAXCAND ? n_cand : RS_MAXCAND;
            if (tid == 0) {
                s_best_d = INFINITY;
                s_best_slot = -1;
                s_exact++;
            }
            __syncthreads();
            for (int ci = 0; ci < nc; ci++) {
                int slot = A.live[cand_list[ci]];
                float lb, ub, d;
                slot_bounds<T>(A, b, fn, slot, lb, ub, d);
                if ((double)lb > s_best_d) continue;  // cannot win (uniform across threads)
                double dx = exact_dist<T>(A, b, slot, sh_slot_of, mlist, scratch);
                if (tid == 0) {
                    int cid = A.s_cid[slot];
                    if (dx < s_best_d || (dx == s_best_d && cid < A.s_cid[s_best_slot])) {
                        s_best_d = dx;
                        s_best_slot = slot;
                    }
                }
                __syncthreads();
            }
            if (tid == 0) {
                if (n_cand > RS_MAXCAND) ctr[C_ERR] = 1;  // candidate overflow (never expected)
                if (s_best_slot >= 0 && s_best_d <= A.T) {
                    s_decision_slot = s_best_slot;
                    s_ub_used = (float)s_best_d * 1.000001f + 1e-30f;
                } else {
                    s_seed = 1;
                }
            }
            __syncthreads();
        }
        // ---- apply (thread 0)
        if (tid == 0) {
            const int64_t c = A.c0 + b;
            const int64_t obj = A.cls_obj[c];
            int slot, rank_m, rank_f;
            if (!s_seed) {
                slot = s_decision_slot;
                rank_m = A.s_size[slot];
                rank_f = A.s_nfeat[slot];
                int nf = rank_f + 1;
                A.s_nfeat[slot] = nf;
                A.s_size[slot] = rank_m + 1;
                A.s_drift[slot] = drift_step(A.s_drift[slot], (double)s_ub_used, nf,
                                             sqrt((double)A.s_cn2[slot]) + (double)A.fnorm[c]);
            } else {
                slot = A.free_stack[--s_nfree];
                int cid = (int)s_next_cid++;
                A.s_cid[slot] = cid;
                A.cid_slot[cid] = slot;
                A.s_nfeat[slot] = 1;
                A.s_size[slot] = 1;
                A.s_drift[slot] = 0.0;
                A.s_cn2[slot] = A.fnorm[c] * A.fnorm[c];
                A.s_snapq[slot] = -1;
                A.s_seedpos[slot] = b;
                A.s_foldpos[slot] = b;
                A.s_pend[slot] = 0;
                A.s_evicted[slot] = 0;
                A.s_odcol[slot] = -1;
                A.s_grp[slot] = -1;
                A.live[s_L] = slot;
                A.live_pos[slot] = s_L;
                s_L++;
                seedlist[s_nseeds++] = slot;
                rank_m = 0;
                rank_f = 0;
                if (A.res_col[b] < 0) {
                    A.s_odcol[slot] = s_nod++;
                    s_need_od = slot;
                }
                if (s_L > A.M) s_need_evict = 1;
            }
            if (A.s_pend[slot] == 0) {  // first member this batch -> dirty
                A.s_didx[slot] = s_ndirty;
                A.dirty[s_ndirty++] = slot;
            }
            A.pend_rank[b] = A.s_pend[slot]++;
            sh_slot_of[b] = slot;
            A.slot_of[b] = slot;
            const int cid = A.s_cid[slot];
            A.cluster_of[obj] = cid;
            A.mrank[obj] = rank_m;
            A.frank[obj] = rank_f;
            s_inserted++;
        }
        __syncthreads();
        // ---- on-demand in-batch column for a seed without a residual column
        if (s_need_od >= 0) {
            const int slot = s_need_od;
            const int col = A.s_odcol[slot];
            const T *fs = (const T *)A.frow[A.c0 + b];
            for (int bb = b + 1 + tid; bb < B; bb += blockDim.x) {
                const T *fo = (const T *)A.frow[A.c0 + bb];
                float tot = 0.f, acc = 0.f;
                for (int k = 0; k < A.D; k++) {
                    float d = (float)fo[k] - (float)fs[k];
                    acc = fmaf(d, d, acc);
                    if ((k & 63) == 63) {
                        tot += acc;
                        acc = 0.f;
                    }
                }
                tot += acc;
                A.dod[(int64_t)col * B + bb] = sqrtf(tot);
            }
        }
        // ---- eviction (clustering.py:139-144)
        if (s_need_evict) {
            if (tid == 0) s_victim_key = 0x7fffffffffffffffLL;
            __syncthreads();
            long long best = 0x7fffffffffffffffLL;
            for (int i = tid; i < s_L; i += blockDim.x) {
                int slot = A.live[i];
                long long key = ((long long)A.s_size[slot] << 32) | (long long)(unsigned)A.s_cid[slot];
                best = key < best ? key : best;
            }
            best = warp_min(best);
            if (lane == 0) atomicMin((unsigned long long *)&s_victim_key, (unsigned long long)best);
            __syncthreads();
            {
                const int vcid = (int)(s_victim_key & 0xffffffffLL);
                for (int i = tid; i < s_L; i += blockDim.x)
                    if (A.s_cid[A.live[i]] == vcid) s_best_slot = A.live[i];
            }
            __syncthreads();
            if (tid == 0) {
                const int vcid = (int)(s_victim_key & 0xffffffffLL);
                const int vslot = s_best_slot;
                int pos = A.live_pos[vslot];
                int last = A.live[s_L - 1];
                A.live[pos] = last;
                A.live_pos[last] = pos;
                s_L--;
                A.s_evicted[vslot] = 1;
                s_any_evicted = 1;
                A.evict_slot[s_nevict] = vslot;
                A.evict_cid[s_nevict] = vcid;
                s_nevict++;
                A.defer_free[s_ndefer++] = vslot;
                if (A.s_pend[vslot] == 0) {  // untouched this batch but needs its final centroid
                    A.s_didx[vslot] = s_ndirty;
                    A.dirty[s_ndirty++] = vslot;
                }
            }
        }
        // ---- dedup members following this object attach to its cluster
        if (tid == 0) {
            int slot = sh_slot_of[b];
            A.s_size[slot] += A.dup_run[A.c0 + b];
        }
        __syncthreads();
        }
        if (tid == 0) {
            A.prof[5] += clock64() - t5;
            A.prof[7]++;
        }
        b = b + 1;
    }

    // ---- epilogue: pending-member CSR for k_fold, snapshot for next batch
    __syncthreads();
    {
        // pending counts of the dirty slots (parallel loads), the largest slot
        // moved first (k_fold gives it its own grid row), offsets by a scan
        int *cnt = mlist;  // mlist + seg_key: 2 * BC ints of scratch, >= the dirty count
        const int nd = s_ndirty;
        int bc = -1, bi = 0;
        for (int i = tid; i < nd; i += blockDim.x) {
            const int c = A.s_pend[A.dirty[i]];
            cnt[i] = c;
            if (c > bc) {
                bc = c;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const int oc = __shfl_xor_sync(0xffffffffu, bc, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oc > bc || (oc == bc && oi < bi)) {
                bc = oc;
                bi = oi;
            }
        }
        if (lane == 0) {
            wsv[wid] = bc;
            wsh[wid] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            int best = 0, bcc = -1;
            for (int w = 0; w < RS_WARPS; w++)
                if (wsv[w] > bcc || (wsv[w] == bcc && wsh[w] < best)) {
                    bcc = wsv[w];
                    best = wsh[w];
                }
            if (best > 0 && nd > 0) {
                const int a0 = A.dirty[0], a1 = A.dirty[best];
                A.dirty[0] = a1;
                A.dirty[best] = a0;
                A.s_didx[a1] = 0;
                A.s_didx[a0] = best;
                const int t = cnt[0];
                cnt[0] = cnt[best];
                cnt[best] = t;
            }
        }
        __syncthreads();
        if (wid == 0) {  // exclusive scan of the counts
            int run = 0;
            for (int i0 = 0; i0 < nd; i0 += 32) {
                const int i = i0 + lane;
                const int c = i < nd ? cnt[i] : 0;
                int x = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (i < nd) {
                    A.dirty_off[i] = run + x - c;
                    cnt[i] = run + x - c;
                }
                run += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) A.dirty_off[nd] = run;
        }
        __syncthreads();
        const int32_t *__restrict__ s_didx = A.s_didx;
        const int32_t *__restrict__ pend_rank = A.pend_rank;
        int32_t *__restrict__ pend_list = A.pend_list;
        for (int bb = tid; bb < B; bb += blockDim.x) {
            const int slot = sh_slot_of[bb];
            const int di = s_didx[slot];
            pend_list[cnt[di] + pend_rank[bb]] = bb;
            A.pend_seg[cnt[di] + pend_rank[bb]] = di;
        }
    }
    for (int q = tid; q < s_L; q += blockDim.x) A.snap_slot[q] = A.live[q];
    __syncthreads();
    if (tid == 0) {
        ctr[C_NLIVE] = s_L;
        ctr[C_NSNAP] = s_L;
        ctr[C_NFREE] = s_nfree;
        ctr[C_NDEFER] = s_ndefer;
        ctr[C_NEVICT_BATCH] = s_nevict;
        ctr[C_NEVICT_TOTAL] += s_nevict;
        ctr[C_NDIRTY] = s_ndirty;
        ctr[C_NOD] = s_nod;
        ctr[C_DC] = s_dc;
        ctr[C_EXACT] = s_exact;
        ctr[C_FAST] = s_fast;
        ctr[C_NEXT_CID] = s_next_cid;
        ctr[C_NINSERTED] = s_inserted;
        ctr[C_LAST_CID] = A.s_cid[sh_slot_of[B - 1]];
        ctr[C_NRES] = 0;
        if (A.h_ring) {  // zero-copy readback (no memcpy in the stream)
            A.h_ring[C_NEXT_CID] = s_next_cid;
            __threadfence_system();
        }
    }
    // the fold re-accumulates ||c||^2 of the slots it refreshes
    for (int i = tid; i < s_ndirty; i += blockDim.x) A.s_cn2[A.dirty[i]] = 0.f;
}


// ---------------------------------------------------------------------------
// K2b fast path: a batch whose every object joins its nearest snapshot
// cluster for certain (the common case once the clusters exist: 799,999 of
// 800,000 objects at C2).  The single-CTA k_resolve above decides the same
// certainty test (pass D) window by window; here the whole batch is one
// window spread over the grid:
//   k_rfast1 (one CTA per 256 objects): hypothesis group = snapshot index of
//     the nearest candidate; stable in-chunk rank (warp match + per-warp
//     group tables), in-chunk prefix sums of the hypothesis upper bounds
//     (fp32, every add rounded up -> an upper bound of the exact sum, as the
//     single-CTA scan) and of the dedup runs; the last CTA to finish scans
//     the chunk tables per group, derives each group's drift bound
//     (drift_avg), the two largest drifts and the fold's dirty order.
//   k_rfast3 (one CTA per 256 objects): per object rank i, prefix P_i, the
//     certainty test ub0 + drift(i) <= T and lbr - max_other_drift > ub;
//     certain objects write their cluster, featured / member / pending rank
//     and pending-list entry; the last CTA commits the slot state -- only if
//     EVERY object was certain, else k_resolve re-runs the batch from the
//     untouched state (it rewrites every per-object output).
// Preconditions (else k_resolve): no residual column (no probable seed),
// snapshot = live set, 0 < L <= RF_MAXG.
// ---------------------------------------------------------------------------
constexpr int RF_T = 256, RF_W = RF_T / 32, RF_MAXG = 256;

__global__ void __launch_bounds__(RF_T) k_rfast1(ResolveArgs A) {
    pdl_enter();
    __shared__ int wc[RF_W][RF_MAXG], wd[RF_W][RF_MAXG];
    __shared__ float wsu[RF_W][RF_MAXG];
    __shared__ int smax[RF_MAXG];
    __shared__ float sh_ub[RF_T];
    __shared__ int sh_dr[RF_T];
    __shared__ int s_last;
    __shared__ double r1[RF_W], r2[RF_W];
    __shared__ int rs[RF_W], scn[RF_W], scf[RF_W];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int64_t *ctr = A.ctr;
    const int B = A.B;
    const int nsnap = (int)ctr[C_NSNAP], L = (int)ctr[C_NLIVE];
    const bool ok = ctr[C_NRES] == 0 && nsnap == L && L > 0 && nsnap <= RF_MAXG && B > 0;
    if (!ok) {
        if (blockIdx.x == 0 && tid == 0) ctr[C_FASTST] = 2;
        return;
    }
    for (int e = tid; e < RF_W * nsnap; e += RF_T) {
        wc[e / nsnap][e % nsnap] = 0;
        wd[e / nsnap][e % nsnap] = 0;
        wsu[e / nsnap][e % nsnap] = 0.f;
    }
    for (int g = tid; g < nsnap; g += RF_T) smax[g] = 0;
    const int p = blockIdx.x * RF_T + tid;
    int g = -1, dr = 0;
    float ub0 = 0.f;
    if (p < B) {
        g = A.sum_q[p];
        if (g < 0 || g >= nsnap) g = -1;
        ub0 = (A.sum_d1[p] + A.sum_e1[p]) * 1.000001f + 1e-30f;
        dr = A.dup_run[A.c0 + p];
    }
    sh_ub[tid] = ub0;
    sh_dr[tid] = dr;
    __syncthreads();
    if (p < B && g < 0) ctr[C_FASTST] = 2;  // no hypothesis: the sequential resolve decides
    const unsigned act = __ballot_sync(0xffffffffu, g >= 0);
    unsigned peers = 0, lower = 0;
    if (g >= 0) {
        peers = __match_any_sync(act, g);
        lower = peers & ((1u << lane) - 1u);
    }
    float Pw = 0.f;
    int Dw = 0;
    for (unsigned m = lower; m; m &= m - 1) {  // earlier same-group lanes, in lane order
        const int l = wid * 32 + __ffs(m) - 1;
        Pw = __fadd_ru(Pw, sh_ub[l]);
        Dw += sh_dr[l];
    }
    const int rw = __popc(lower);
    if (g >= 0) {
        if ((peers >> lane) == 1u) {  // highest lane of its group writes the warp totals
            wc[wid][g] = rw + 1;
            wsu[wid][g] = __fadd_ru(Pw, ub0);
            wd[wid][g] = Dw + dr;
        }
        atomicMax(&smax[g], __float_as_int(ub0));  // ub0 > 0: int order = float order
    }
    __syncthreads();
    for (int gg = tid; gg < nsnap; gg += RF_T) {  // exclusive scan over warps, chunk totals
        int c = 0, d = 0;
        float su = 0.f;
        for (int w = 0; w < RF_W; w++) {
            const int cw = wc[w][gg], dw = wd[w][gg];
            const float sw = wsu[w][gg];
            wc[w][gg] = c;
            wd[w][gg] = d;
            wsu[w][gg] = su;
            c += cw;
            d += dw;
            su = __fadd_ru(su, sw);
        }
        const int idx = blockIdx.x * RF_MAXG + gg;
        A.f_ccnt[idx] = c;
        A.f_cdup[idx] = d;
        A.f_csum[idx] = su;
        A.f_cmax[idx] = __int_as_float(smax[gg]);
    }
    __syncthreads();
    if (g >= 0) {
        A.f_rank[p] = wc[wid][g] + rw;
        A.f_P[p] = __fadd_ru(wsu[wid][g], Pw);
        A.f_dup[p] = wd[wid][g] + Dw;
    }
    // last CTA: per group scan over the chunks -> bases, totals, drift bounds
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd((unsigned long long *)&ctr[C_FDONE], 1ull) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int nch = gridDim.x;
    int c = 0, d = 0;
    float su = 0.f, mx = 0.f, drift = 0.f;
    const int gg = tid;  // nsnap <= RF_MAXG = RF_T: one group per thread
    // the group's slot state, fetched before the chunk scan
    int g_sl = 0, g_nf = 0, g_cid = 0, g_size = 0;
    float g_cn2 = 0.f;
    double g_sdev = 0.0;
    if (gg < nsnap) {
        g_sl = A.snap_slot[gg];
        g_cn2 = A.s_cn2[g_sl];
        g_sdev = A.s_sdev[g_sl];
        g_nf = A.s_nfeat[g_sl];
        g_cid = A.s_cid[g_sl];
        g_size = A.s_size[g_sl];
    }
    if (gg < nsnap) {
        // chunk totals -> exclusive bases; 8 chunks' loads in flight before
        // the dependent scan (the stores would otherwise serialise them)
        for (int k0 = 0; k0 < nch; k0 += 8) {
            int ck[8], dk[8];
            float sk[8], mk[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int idx = (k0 + u) * RF_MAXG + gg;
                const bool in = k0 + u < nch;
                ck[u] = in ? __ldcg(A.f_ccnt + idx) : 0;
                dk[u] = in ? __ldcg(A.f_cdup + idx) : 0;
                sk[u] = in ? __ldcg(A.f_csum + idx) : 0.f;
                mk[u] = in ? __ldcg(A.f_cmax + idx) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                if (k0 + u >= nch) break;
                const int idx = (k0 + u) * RF_MAXG + gg;
                A.f_ccnt[idx] = c;
                A.f_cdup[idx] = d;
                A.f_csum[idx] = su;
                c += ck[u];
                d += dk[u];
                su = __fadd_ru(su, sk[u]);
                mx = fmaxf(mx, mk[u]);
            }
        }
        const float cn = sqrtf(g_cn2) * 1.00001f;
        const float d0 = __double2float_ru(g_sdev);  // k_resolve's prologue: s_drift = s_sdev
        drift = c > 0 ? drift_avg(d0, g_nf, su, c, cn, mx) : d0;
        A.f_gi[gg * 8 + 0] = c;
        A.f_gi[gg * 8 + 1] = d;
        A.f_gi[gg * 8 + 4] = g_sl;  // the group's slot state for k_rfast3 (one round of loads)
        A.f_gi[gg * 8 + 5] = g_nf;
        A.f_gi[gg * 8 + 6] = g_cid;
        A.f_gi[gg * 8 + 7] = g_size;
        A.f_gf[gg * 4 + 0] = drift;
        A.f_gf[gg * 4 + 1] = mx;
        A.f_gf[gg * 4 + 2] = cn;
        A.f_gf[gg * 4 + 3] = d0;
    }
    // the two largest end-of-batch drifts over the live (= snapshot) slots
    double m1 = gg < nsnap ? (double)drift : -1.0, m2 = -1.0;
    int m1s = gg < nsnap ? gg : -1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double o1 = __shfl_xor_sync(0xffffffffu, m1, o), o2 = __shfl_xor_sync(0xffffffffu, m2, o);
        const int os = __shfl_xor_sync(0xffffffffu, m1s, o);
        if (o1 > m1) {
            m2 = fmax(m1, o2);
            m1 = o1;
            m1s = os;
        } else {
            m2 = fmax(m2, o1);
        }
    }
    if (lane == 0) {
        r1[wid] = m1;
        r2[wid] = m2;
        rs[wid] = m1s;
    }
    // dirty order: the group with the most members first (k_fold gives it its
    // own grid row), then the others in snapshot order; offsets = scan of counts
    int bc = gg < nsnap ? c : -1, bi = gg;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oc > bc || (oc == bc && oi < bi)) {
            bc = oc;
            bi = oi;
        }
    }
    if (lane == 0) {
        scn[wid] = bc;
        scf[wid] = bi;
    }
    __syncthreads();
    if (tid == 0) {
        double a1 = r1[0], a2 = r2[0];
        int as = rs[0];
        int best = scf[0], bcc = scn[0];
        for (int w = 1; w < RF_W; w++) {
            if (r1[w] > a1) {
                a2 = fmax(a1, r2[w]);
                a1 = r1[w];
                as = rs[w];
            } else {
                a2 = fmax(a2, r1[w]);
            }
            if (scn[w] > bcc || (scn[w] == bcc && scf[w] < best)) {
                bcc = scn[w];
                best = scf[w];
            }
        }
        A.f_gd[0] = a1 < 0 ? 0.0 : a1;
        A.f_gd[1] = a2 < 0 ? 0.0 : a2;
        A.f_gd[2] = (double)as;
        A.f_gd[3] = (double)best;
        A.f_gd[4] = (double)bcc;
    }
    __syncthreads();
    const int best = (int)A.f_gd[3], bcc = (int)A.f_gd[4];
    const bool fl = gg < nsnap && c > 0 && gg != best;
    const int cv = fl ? c : 0;
    int xf = fl ? 1 : 0, xc = cv;  // inclusive warp scans of (dirty flag, count)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int yf = __shfl_up_sync(0xffffffffu, xf, o), yc = __shfl_up_sync(0xffffffffu, xc, o);
        if (lane >= o) {
            xf += yf;
            xc += yc;
        }
    }
    __syncthreads();
    if (lane == 31) {
        scf[wid] = xf;
        scn[wid] = xc;
    }
    __syncthreads();
    int bf = 0, bcn = 0;
    for (int w = 0; w < wid; w++) {
        bf += scf[w];
        bcn += scn[w];
    }
    if (gg < nsnap) {
        const bool has = bcc > 0;  // the largest group is dirty[0] when any object joined
        if (gg == best && c > 0) {
            A.f_gi[gg * 8 + 2] = 0;
            A.f_gi[gg * 8 + 3] = 0;
        } else if (fl) {
            A.f_gi[gg * 8 + 2] = (has ? 1 : 0) + bf + xf - 1;
            A.f_gi[gg * 8 + 3] = (has ? bcc : 0) + bcn + xc - cv;
        } else {
            A.f_gi[gg * 8 + 2] = -1;
            A.f_gi[gg * 8 + 3] = 0;
        }
    }
    if (tid == 0) ctr[C_FDONE] = 0;
}

__global__ void __launch_bounds__(RF_T) k_rfast3(ResolveArgs A) {
    pdl_enter();
    __shared__ int s_last, s_fail;
    const int tid = threadIdx.x;
    int64_t *ctr = A.ctr;
    const bool declined = ctr[C_FASTST] == 2;  // k_rfast1 declined
    const int B = A.B;
    const double md1 = A.f_gd[0], md2 = A.f_gd[1];
    const int md1g = (int)A.f_gd[2];
    if (tid == 0) s_fail = 0;
    __syncthreads();
    const int p = blockIdx.x * RF_T + tid;
    if (p < B && !declined) {
        const int g = A.sum_q[p];
        const int idx = blockIdx.x * RF_MAXG + g;
        const int i = A.f_ccnt[idx] + A.f_rank[p];
        const float P = __fadd_ru(A.f_csum[idx], A.f_P[p]);
        const int sl = A.f_gi[g * 8 + 4];
        const int nf0 = A.f_gi[g * 8 + 5];
        const float ub0 = (A.sum_d1[p] + A.sum_e1[p]) * 1.000001f + 1e-30f;
        const double ub =
            (double)ub0 + (double)drift_avg(A.f_gf[g * 4 + 3], nf0, P, i, A.f_gf[g * 4 + 2], A.f_gf[g * 4 + 1]);
        const float lbr = A.sum_lbr[p];
        const float lbr2 = lbr - fabsf(lbr) * 1e-6f - 1e-30f;
        const double md = g == md1g ? md2 : md1;
        const double lbo = (double)lbr2 - md * 1.000001;
        if (lbo > ub && ub <= A.T) {
            const int64_t obj = A.cls_obj[A.c0 + p];
            A.cluster_of[obj] = A.f_gi[g * 8 + 6];
            A.mrank[obj] = A.f_gi[g * 8 + 7] + i + A.f_cdup[idx] + A.f_dup[p];
            A.frank[obj] = nf0 + i;
            A.pend_rank[p] = i;
            A.slot_of[p] = sl;
            A.pend_list[A.f_gi[g * 8 + 3] + i] = p;
            A.pend_seg[A.f_gi[g * 8 + 3] + i] = A.f_gi[g * 8 + 2];
        } else {
            s_fail = 1;
        }
    }
    __syncthreads();
    if (tid == 0 && s_fail) ctr[C_FASTST] = 2;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd((unsigned long long *)&ctr[C_FDONE], 1ull) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (tid == 0) ctr[C_FDONE] = 0;
    if (__ldcg(&ctr[C_FASTST]) == 2) return;  // some object needs the sequential resolve
    // commit: k_resolve's prologue (recycle deferred slots, reset snapshot
    // fields), the groups' slot state, the fold's dirty CSR, the counters
    const int nsnap = (int)ctr[C_NSNAP], L = (int)ctr[C_NLIVE];
    const int gg = tid;
    int nd = 0;
    if (gg < nsnap) {
        const int sl = A.f_gi[gg * 8 + 4];
        const int c = A.f_gi[gg * 8 + 0];
        A.s_snapq[sl] = gg;
        A.s_seedpos[sl] = -1;
        A.s_foldpos[sl] = 0;
        A.s_odcol[sl] = -1;
        if (c > 0) {
            const int di = A.f_gi[gg * 8 + 2];
            A.s_drift[sl] = (double)A.f_gf[gg * 4 + 0];
            A.s_nfeat[sl] = A.f_gi[gg * 8 + 5] + c;
            A.s_size[sl] = A.f_gi[gg * 8 + 7] + c + A.f_gi[gg * 8 + 1];
            A.s_pend[sl] = c;
            A.s_didx[sl] = di;
            A.dirty[di] = sl;
            A.dirty_off[di] = A.f_gi[gg * 8 + 3];
            A.s_cn2[sl] = 0.f;  // the fold re-accumulates ||c||^2
        } else {
            A.s_drift[sl] = A.s_sdev[sl];
            A.s_pend[sl] = 0;
        }
    }
    const unsigned long long has = __ballot_sync(0xffffffffu, gg < nsnap && A.f_gi[gg * 8 + 0] > 0);
    __shared__ int s_nd;
    if (tid == 0) s_nd = 0;
    __syncthreads();
    if ((tid & 31) == 0) atomicAdd(&s_nd, __popc((unsigned)has));
    __syncthreads();
    nd = s_nd;
    if (tid == 0) {
        int nfree = (int)ctr[C_NFREE];
        const int ndf = (int)ctr[C_NDEFER];
        for (int k = 0; k < ndf; k++) A.free_stack[nfree++] = A.defer_free[k];
        A.dirty_off[nd] = B;
        ctr[C_NFREE] = nfree;
        ctr[C_NDEFER] = 0;
        ctr[C_NEVICT_BATCH] = 0;
        ctr[C_NDIRTY] = nd;
        ctr[C_NOD] = 0;
        ctr[C_NSNAP] = L;
        ctr[C_DC] += (int64_t)L * B;
        ctr[C_FAST] += B;
        ctr[C_NINSERTED] += B;
        ctr[C_LAST_CID] = A.f_gi[A.sum_q[B - 1] * 8 + 6];  // the fast path creates no cluster
        ctr[C_FASTB] += 1;
        if (A.h_ring) {
            A.h_ring[C_NEXT_CID] = ctr[C_NEXT_CID];
            __threadfence_system();
        }
        ctr[C_FASTST] = 1;
    }
}

// ---------------------------------------------------------------------------
// K2c: fold the batch's members into the float64 sums (stream order) and
// refresh the FP32 snapshot; record final centroids of evicted clusters.
// grid (ceil(D/256), ndirty)
// ---------------------------------------------------------------------------

// One CTA per (dirty slot, FD-dimension slice).  A slot's members must be
// added in stream order (float64 rounding is order dependent), so each
// dimension is one dependent dadd chain; what limits the chain is how fast
// member rows arrive.  Warp-specialised pipeline: warp 0 (lane = dimension)
// walks the chain out of a FOLD_NS-buffer shared-memory ring; producer warp
// w (1..FOLD_NS) owns buffer w-1 and fills it with every FOLD_NS-th stage of
// R rows x FD dims (gather the rows' pointers, cp.async the slices, wait,
// then publish with an mbarrier arrive).  So FOLD_NS * R rows are in flight
// for the dominant cluster of a Zipf stream, which owns most of a batch.
constexpr int FD = 32, FOLD_NS = 6, FOLD_THREADS = 32 * (1 + FOLD_NS);
template <typename T>
constexpr int fold_rows() { return sizeof(T) == 4 ? 64 : 32; }  // 8 KB per stage (32 rows: slower, 128: later first stage)
template <typename T>
constexpr size_t fold_smem() { return (size_t)FOLD_NS * fold_rows<T>() * FD * sizeof(T); }

__device__ __forceinline__ void cp_async_el(uint32_t dst, const void *src, bool ok, int bytes) {
    if (bytes == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void fbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void fbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void fbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nFW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra FW_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
        "r"(parity)
        : "memory");
}

// Chain descriptor: what k_tfold hands the lagged exact chain for one batch
// (double buffered: batch b uses buffer b % 2).  meta rows: slot, featured
// count after the batch, fold position, seed position, evicted, cluster id,
// size.  rows: the members to add in stream order (nullptr: already in S --
// folded by the resolve's exact path).
enum CdMeta { CD_SLOT = 0, CD_NFEAT, CD_FP, CD_SP, CD_EV, CD_CID, CD_SIZE, CD_NMETA = 8 };
struct ChainDesc {
    const int64_t *nd;
    const int32_t *meta;  // [CD_NMETA][ldm]
    int ldm;
    const int32_t *off;
    const char *const *rows;
};

// ---------------------------------------------------------------------------
// K2c': snapshot tree fold (main stream, right after the resolve).  The next
// batch's screen needs the FP32 snapshot of every moved centroid, not the
// reference's sequential float64 sum: each dirty slot's rows are added in a
// fixed tree order into S_tree (float64), C32 = fp32(S_tree / n), and the
// distance between that centroid and the reference's exact one is bounded
// (Higham: any summation order of n terms is within gamma_n sum |x_i| of the
// real sum, coordinate-wise, so the two float64 sums differ by at most
// 2 gamma_n sum_i ||x_i|| in 2-norm) and handed to the resolve as the slot's
// starting drift.  The reference's own sum (clustering.py:56-59) is still
// computed bit for bit -- by the chain below, one batch behind, off the
// critical path.  This kernel also writes the chain's descriptor.
// grid (ceil(D/32), rows): row 0 takes dirty[0] (the largest slot), the
// others stride over the rest; 8 warps x 4 interleaved accumulators per
// 32-column slice, combined in a fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int TF_T = 512, TF_W = TF_T / 32, TF_C = 128, TF_SPLIT = 16;

template <typename T>
__global__ void __launch_bounds__(TF_T) k_tfold(int D, int64_t c0, int B, const int64_t *__restrict__ ctr,
                                                const int32_t *__restrict__ dirty, const int32_t *__restrict__ dirty_off,
                                                const int32_t *__restrict__ pend_list, const char *const *__restrict__ frow,
                                                const float *__restrict__ fnorm, const int32_t *__restrict__ s_nfeat,
                                                const int32_t *__restrict__ s_foldpos, const int32_t *__restrict__ s_seedpos,
                                                const int32_t *__restrict__ s_evicted, const int32_t *__restrict__ s_cid,
                                                const int32_t *__restrict__ s_size, double *__restrict__ S_tree,
                                                float *__restrict__ C32, float *__restrict__ s_cn2,
                                                double *__restrict__ s_abs, double *__restrict__ s_sdev,
                                                float *__restrict__ tf_cn2, int32_t *__restrict__ tf_cnt,
                                                double *__restrict__ tf_part, int32_t *__restrict__ tf_bcnt,
                                                int64_t *__restrict__ cd_nd, int32_t *__restrict__ cd_meta, int ldm,
                                                int32_t *__restrict__ cd_off, const char **__restrict__ cd_rows) {
    pdl_enter();
    __shared__ double part[TF_W][TF_C];
    __shared__ double s_fn[TF_W];
    __shared__ float s_c2[TF_W];
    __shared__ int s_last;
    const int nd = (int)ctr[C_NDIRTY];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int gx = gridDim.x, x = blockIdx.x, y = blockIdx.y;
    if (x == 0 && y == 0 && tid == 0) {
        *cd_nd = nd;
        cd_off[nd] = dirty_off[nd];
    }
    // rows y < TF_SPLIT share dirty[0] (the largest slot: the resolve puts it
    // first) in row chunks, combined in chunk order; the other rows take the
    // remaining slots whole
    const bool split = y < TF_SPLIT;
    const int dstart = split ? 0 : 1 + (y - TF_SPLIT);
    const int dstep = split ? nd : (int)gridDim.y - TF_SPLIT;
    for (int di = dstart; di < nd; di += dstep) {
        const int slot = dirty[di];
        const int j0 = dirty_off[di], j1 = dirty_off[di + 1];
        const int ra = split ? j0 + (int)((int64_t)(j1 - j0) * y / TF_SPLIT) : j0;
        const int rb = split ? j0 + (int)((int64_t)(j1 - j0) * (y + 1) / TF_SPLIT) : j1;
        const int fp = s_foldpos[slot], sp = s_seedpos[slot], ev = s_evicted[slot];
        const int n = s_nfeat[slot];
        if (x == 0) {  // the chain's descriptor: this CTA's rows, and the slot's meta
            for (int j = ra + tid; j < rb; j += TF_T) {
                const int p = pend_list[j];
                cd_rows[j] = p >= fp ? frow[c0 + p] : nullptr;
            }
            if (tid == 0 && (!split || y == 0)) {
                cd_off[di] = j0;
                cd_meta[CD_SLOT * ldm + di] = slot;
                cd_meta[CD_NFEAT * ldm + di] = n;
                cd_meta[CD_FP * ldm + di] = fp;
                cd_meta[CD_SP * ldm + di] = sp;
                cd_meta[CD_EV * ldm + di] = ev;
                cd_meta[CD_CID * ldm + di] = s_cid[slot];
                cd_meta[CD_SIZE * ldm + di] = s_size[slot];
            }
        }
        if (ev) continue;  // evicted: no snapshot (its exact centroid comes from the chain)
        const bool fresh = sp >= 0;  // seeded in this batch: S_tree starts empty
        // warp w sums the 32-row groups w, w + 16, ... of [ra, rb): the group's
        // row pointers are gathered by its lanes first, so 8 rows' loads are
        // in flight at once; lane l owns columns x*128 + l + 32 i
        double acc[4][2];
#pragma unroll
        for (int i = 0; i < 4; i++) acc[i][0] = acc[i][1] = 0.0;
        double fsum = 0.0;
        for (int g0 = ra + 32 * wid; g0 < rb; g0 += 32 * TF_W) {
            const int jl = g0 + lane;
            const T *ptr = nullptr;
            if (jl < rb) {
                const int p = pend_list[jl];
                ptr = (const T *)frow[c0 + p];
                if (x == 0) fsum += (double)fnorm[c0 + p];
            }
            const int nr = min(32, rb - g0);
#pragma unroll 8
            for (int r = 0; r < nr; r++) {
                const T *row = (const T *)__shfl_sync(0xffffffffu, (unsigned long long)ptr, r);
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int col = x * TF_C + lane + 32 * i;
                    if (col < D) acc[i][r & 1] = dadd(acc[i][r & 1], to_d(row[col]));
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) part[wid][lane + 32 * i] = dadd(acc[i][0], acc[i][1]);
        if (x == 0) {
            fsum = warp_sum(fsum);
            if (lane == 0) s_fn[wid] = fsum;
        }
        __syncthreads();
        double t = 0.0, fs = 0.0;
        const int col = x * TF_C + tid;
        if (tid < TF_C) {
            t = part[0][tid];
#pragma unroll
            for (int w = 1; w < TF_W; w++) t = dadd(t, part[w][tid]);
        }
        if (x == 0 && tid == 0)
            for (int w = 0; w < TF_W; w++) fs += s_fn[w];
        bool finish = true;
        if (split) {  // publish this chunk; the slice's last chunk combines them in order
            if (tid < TF_C && col < D) tf_part[(int64_t)y * D + col] = t;
            if (x == 0 && tid == 0) tf_part[(int64_t)TF_SPLIT * D + y] = fs;
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = atomicAdd(&tf_bcnt[x], 1) == TF_SPLIT - 1;
            __syncthreads();
            finish = s_last;
            if (finish) {
                __threadfence();
                if (tid < TF_C && col < D) {
                    t = __ldcg(&tf_part[col]);
                    for (int q = 1; q < TF_SPLIT; q++) t = dadd(t, __ldcg(&tf_part[(int64_t)q * D + col]));
                }
                if (x == 0 && tid == 0) {
                    fs = 0.0;
                    for (int q = 0; q < TF_SPLIT; q++) fs += __ldcg(&tf_part[(int64_t)TF_SPLIT * D + q]);
                }
                if (tid == 0) tf_bcnt[x] = 0;
            }
        }
        if (finish) {
            float c2 = 0.f;
            if (tid < TF_C && col < D) {
                const double sum = fresh ? t : dadd(S_tree[(int64_t)slot * D + col], t);
                S_tree[(int64_t)slot * D + col] = sum;
                const float c32 = (float)ddiv(sum, (double)n);
                C32[(int64_t)slot * D + col] = c32;
                c2 = c32 * c32;
            }
            c2 = warp_sum(c2);
            if (lane == 0) s_c2[wid] = c2;
            __syncthreads();
            if (tid == 0) {
                float cs = 0.f;
                for (int w = 0; w < TF_C / 32; w++) cs += s_c2[w];
                tf_cn2[(int64_t)di * gx + x] = cs;
                // fp32 norms: relative error < 1e-6, rounded up
                if (x == 0) s_abs[slot] = (fresh ? 0.0 : s_abs[slot]) + fs * (1.0 + 1e-5);
                __threadfence();
                s_last = atomicAdd(&tf_cnt[di], 1) == gx - 1;
            }
            __syncthreads();
            if (s_last && tid == 0) {  // last slice: ||C32||^2 in slice order, the drift bound
                __threadfence();
                float cs = 0.f;
                for (int q = 0; q < gx; q++) cs += __ldcg(&tf_cn2[(int64_t)di * gx + q]);
                s_cn2[slot] = cs;
                const double u = 1.1102230246251565e-16, nn = (double)n;
                const double gam = nn * u / (1.0 - nn * u);
                const double sa = __ldcg(&s_abs[slot]);
                s_sdev[slot] = (2.0 * gam * sa / nn + 4.0 * u * sqrt((double)cs) * 1.01) * 1.01 + 1e-300;
                tf_cnt[di] = 0;
            }
        }
        __syncthreads();
    }
}

// K2c' (current): the snapshot tree fold in two load-balanced passes.
//   k_tfold_a: CTA (slice x of 512 columns, chunk c of TF3_R pending rows),
//     one column per thread: the chunk's rows are summed in row order per
//     "piece" (the part of one dirty slot's row range inside the chunk; a new
//     piece starts at the chunk start and at every slot boundary) and each
//     piece's float64 column sums go to P[piece start row] (its fp32-norm sum
//     to PF).  Row pointers and piece starts are staged in shared memory; 16
//     row loads per thread are in flight.
//   k_tfold_b: CTA (slice x, dirty slot di): the slot's pieces (start j0, then
//     every chunk boundary inside [j0, j1)) are added in row order, then the
//     slot's S_tree / C32 / norms / drift bound are refreshed as in k_tfold.
// Every order is fixed (deterministic); whatever the order, the float64 sum
// is within the Higham bound of the reference's sequential sum (s_sdev).
// ---------------------------------------------------------------------------
constexpr int TF3_T = 512, TF3_R = 64;

template <typename T>
__global__ void __launch_bounds__(TF3_T) k_tfold_a(int D, int64_t c0, int Btot, const int32_t *__restrict__ dirty,
                                                   const int32_t *__restrict__ pend_list,
                                                   const int32_t *__restrict__ pend_seg,
                                                   const char *const *__restrict__ frow,
                                                   const float *__restrict__ fnorm,
                                                   const int32_t *__restrict__ s_foldpos, double *__restrict__ P,
                                                   double *__restrict__ PF, const char **__restrict__ cd_rows) {
    pdl_enter();
    __shared__ const T *s_row[TF3_R];
    __shared__ float s_fn[TF3_R];
    __shared__ int s_start[TF3_R], s_p[TF3_R], s_seg[TF3_R];
    const int tid = threadIdx.x, x = blockIdx.x, c = blockIdx.y;
    const int cs = c * TF3_R, nr = min(TF3_R, Btot - cs);
    if (nr <= 0) return;
    if (tid < nr) {  // two rounds of independent loads per row
        const int j = cs + tid;
        const int p = pend_list[j], sg = pend_seg[j];
        const int sp = tid > 0 ? pend_seg[j - 1] : -1;
        s_row[tid] = (const T *)frow[c0 + p];
        s_fn[tid] = fnorm[c0 + p];
        s_start[tid] = (tid == 0 || sp != sg) ? 1 : 0;
        s_p[tid] = p;
        s_seg[tid] = sg;
    }
    __syncthreads();
    const int col = x * TF3_T + tid;
    if (col < D) {
        double acc = 0.0;
        int ps = 0;
        for (int r0 = 0; r0 < nr; r0 += 16) {
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; u++) v[u] = r0 + u < nr ? to_d(__ldg(s_row[r0 + u] + col)) : 0.0;
#pragma unroll
            for (int u = 0; u < 16; u++) {
                const int r = r0 + u;
                if (r < nr) {
                    if (s_start[r]) {
                        if (r > 0) P[(int64_t)(cs + ps) * D + col] = acc;
                        acc = v[u];
                        ps = r;
                    } else {
                        acc = dadd(acc, v[u]);
                    }
                }
            }
        }
        P[(int64_t)(cs + ps) * D + col] = acc;
    }
    if (x == 0) {
        if (tid == 0) {  // the pieces' fp32-norm sums
            double f = 0.0;
            int ps = 0;
            for (int r = 0; r < nr; r++) {
                if (s_start[r] && r > 0) {
                    PF[cs + ps] = f;
                    f = 0.0;
                    ps = r;
                }
                f += (double)s_fn[r];
            }
            PF[cs + ps] = f;
        }
        // the lagged chain's rows (nullptr: already folded by the exact path)
        if (tid < nr) cd_rows[cs + tid] = s_p[tid] >= s_foldpos[dirty[s_seg[tid]]] ? (const char *)s_row[tid] : nullptr;
    }
}

// k_tfold_a for fp32 rows with 16-byte alignment: 128 threads per CTA, 4
// adjacent columns per thread (float4 loads, 16 rows in flight = 256 B per
// thread), same pieces, same per-column row order, same P / PF / cd_rows.
constexpr int TF4_T = 128;
__global__ void __launch_bounds__(TF4_T, 4) k_tfold_a4(int D, int64_t c0, int Btot, const int32_t *__restrict__ dirty,
                                                   const int32_t *__restrict__ pend_list,
                                                   const int32_t *__restrict__ pend_seg,
                                                   const char *const *__restrict__ frow,
                                                   const float *__restrict__ fnorm,
                                                   const int32_t *__restrict__ s_foldpos, double *__restrict__ P,
                                                   double *__restrict__ PF, const char **__restrict__ cd_rows) {
    pdl_enter();
    __shared__ const float *s_row[TF3_R];
    __shared__ float s_fn[TF3_R];
    __shared__ int s_start[TF3_R], s_p[TF3_R], s_seg[TF3_R];
    const int tid = threadIdx.x, x = blockIdx.x, c = blockIdx.y;
    const int cs = c * TF3_R, nr = min(TF3_R, Btot - cs);
    if (nr <= 0) return;
    if (tid < nr) {
        const int j = cs + tid;
        const int p = pend_list[j], sg = pend_seg[j];
        const int sp = tid > 0 ? pend_seg[j - 1] : -1;
        s_row[tid] = (const float *)frow[c0 + p];
        s_fn[tid] = fnorm[c0 + p];
        s_start[tid] = (tid == 0 || sp != sg) ? 1 : 0;
        s_p[tid] = p;
        s_seg[tid] = sg;
    }
    __syncthreads();
    const int col = x * (4 * TF4_T) + 4 * tid;
    if (col < D) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        int ps = 0;
        auto flush = [&](int at) {
            double2 *dst = (double2 *)(P + (int64_t)(cs + at) * D + col);
            dst[0] = make_double2(acc[0], acc[1]);
            dst[1] = make_double2(acc[2], acc[3]);
        };
        for (int r0 = 0; r0 < nr; r0 += 16) {
            float4 v[16];
#pragma unroll
            for (int u = 0; u < 16; u++)
                v[u] = r0 + u < nr ? __ldg((const float4 *)(s_row[r0 + u] + col)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 16; u++) {
                const int r = r0 + u;
                if (r < nr) {
                    if (s_start[r]) {
                        if (r > 0) flush(ps);
                        acc[0] = (double)v[u].x;
                        acc[1] = (double)v[u].y;
                        acc[2] = (double)v[u].z;
                        acc[3] = (double)v[u].w;
                        ps = r;
                    } else {
                        acc[0] = dadd(acc[0], (double)v[u].x);
                        acc[1] = dadd(acc[1], (double)v[u].y);
                        acc[2] = dadd(acc[2], (double)v[u].z);
                        acc[3] = dadd(acc[3], (double)v[u].w);
                    }
                }
            }
        }
        flush(ps);
    }
    if (x == 0) {
        if (tid == 0) {  // the pieces' fp32-norm sums
            double f = 0.0;
            int ps = 0;
            for (int r = 0; r < nr; r++) {
                if (s_start[r] && r > 0) {
                    PF[cs + ps] = f;
                    f = 0.0;
                    ps = r;
                }
                f += (double)s_fn[r];
            }
            PF[cs + ps] = f;
        }
        if (tid < nr) cd_rows[cs + tid] = s_p[tid] >= s_foldpos[dirty[s_seg[tid]]] ? (const char *)s_row[tid] : nullptr;
    }
}

__global__ void __launch_bounds__(TF3_T) k_tfold_b(
    int D, const int64_t *__restrict__ ctr, const int32_t *__restrict__ dirty, const int32_t *__restrict__ dirty_off,
    const int32_t *__restrict__ s_nfeat, const int32_t *__restrict__ s_foldpos, const int32_t *__restrict__ s_seedpos,
    const int32_t *__restrict__ s_evicted, const int32_t *__restrict__ s_cid, const int32_t *__restrict__ s_size,
    const double *__restrict__ P, const double *__restrict__ PF, double *__restrict__ S_tree, float *__restrict__ C32,
    float *__restrict__ s_cn2, double *__restrict__ s_abs, double *__restrict__ s_sdev, float *__restrict__ tf_cn2,
    int32_t *__restrict__ tf_cnt, int64_t *__restrict__ cd_nd, int32_t *__restrict__ cd_meta, int ldm,
    int32_t *__restrict__ cd_off) {
    pdl_enter();
    __shared__ float s_c2[TF3_T / 32];
    __shared__ int s_last;
    const int nd = (int)ctr[C_NDIRTY];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int x = blockIdx.x, gx = gridDim.x;
    if (x == 0 && blockIdx.y == 0 && tid == 0) {
        *cd_nd = nd;
        cd_off[nd] = dirty_off[nd];
    }
    for (int di = blockIdx.y; di < nd; di += gridDim.y) {
    const int j0 = dirty_off[di], j1 = dirty_off[di + 1];
    const int slot = dirty[di];
    const int sp = s_seedpos[slot], ev = s_evicted[slot];
    if (x == 0 && tid == 0) {  // the lagged chain's descriptor
        cd_off[di] = j0;
        cd_meta[CD_SLOT * ldm + di] = slot;
        cd_meta[CD_NFEAT * ldm + di] = s_nfeat[slot];
        cd_meta[CD_FP * ldm + di] = s_foldpos[slot];
        cd_meta[CD_SP * ldm + di] = sp;
        cd_meta[CD_EV * ldm + di] = ev;
        cd_meta[CD_CID * ldm + di] = s_cid[slot];
        cd_meta[CD_SIZE * ldm + di] = s_size[slot];
    }
    if (ev) continue;  // evicted: no snapshot (its exact centroid comes from the chain)
    const int np = j1 > j0 ? (j1 - 1) / TF3_R - j0 / TF3_R + 1 : 0;
    auto pstart = [&](int k) { return k == 0 ? j0 : (j0 / TF3_R + k) * TF3_R; };
    const int col = x * TF3_T + tid;
    double t = 0.0;
    if (col < D) {
        for (int k0 = 0; k0 < np; k0 += 16) {
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; u++) v[u] = k0 + u < np ? __ldcg(P + (int64_t)pstart(k0 + u) * D + col) : 0.0;
#pragma unroll
            for (int u = 0; u < 16; u++)
                if (k0 + u < np) t = (k0 + u == 0) ? v[u] : dadd(t, v[u]);
        }
    }
    double fs = 0.0;
    if (x == 0 && wid == 0) {
        for (int k = lane; k < np; k += 32) fs += __ldcg(PF + pstart(k));
        fs = warp_sum(fs);
    }
    const bool fresh = sp >= 0;  // seeded in this batch: S_tree starts empty
    const int n = s_nfeat[slot];
    float c2 = 0.f;
    if (col < D) {
        const double sum = fresh ? t : dadd(S_tree[(int64_t)slot * D + col], t);
        S_tree[(int64_t)slot * D + col] = sum;
        const float c32 = (float)ddiv(sum, (double)n);
        C32[(int64_t)slot * D + col] = c32;
        c2 = c32 * c32;
    }
    c2 = warp_sum(c2);
    if (lane == 0) s_c2[wid] = c2;
    __syncthreads();
    if (tid == 0) {
        float cs2 = 0.f;
        for (int w = 0; w < TF3_T / 32; w++) cs2 += s_c2[w];
        tf_cn2[(int64_t)di * gx + x] = cs2;
        // fp32 norms: relative error < 1e-6, rounded up
        if (x == 0) s_abs[slot] = (fresh ? 0.0 : s_abs[slot]) + fs * (1.0 + 1e-5);
        __threadfence();
        s_last = atomicAdd(&tf_cnt[di], 1) == gx - 1;
    }
    __syncthreads();
    if (s_last && tid == 0) {  // last slice: ||C32||^2 in slice order, the drift bound
        __threadfence();
        float cs2 = 0.f;
        for (int q = 0; q < gx; q++) cs2 += __ldcg(&tf_cn2[(int64_t)di * gx + q]);
        s_cn2[slot] = cs2;
        const double u = 1.1102230246251565e-16, nn = (double)n;
        const double gam = nn * u / (1.0 - nn * u);
        const double sa = __ldcg(&s_abs[slot]);
        s_sdev[slot] = (2.0 * gam * sa / nn + 4.0 * u * sqrt((double)cs2) * 1.01) * 1.01 + 1e-300;
        tf_cnt[di] = 0;
    }
    __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K2c: the reference's float64 running sums, bit for bit (clustering.py:56-59),
// one batch behind on the engine's second stream: for each slot of the
// batch's chain descriptor, its members are added in stream order, and an
// evicted slot's final centroid (S / n, sealed at eviction) is recorded.
// The resolve of the next batch waits for this only where it reads S (its
// exact path); the screen and the fast path never do.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(FOLD_THREADS) k_fold(int D, ChainDesc cd, double *__restrict__ S,
                                                      double *__restrict__ fcent, int32_t *__restrict__ cl_nfeat,
                                                      int32_t *__restrict__ cl_size, long long *__restrict__ fprof,
                                                      unsigned int *__restrict__ done_ctas,
                                                      unsigned long long *__restrict__ chain_epoch) {
    constexpr int R = fold_rows<T>();
    extern __shared__ __align__(16) unsigned char fold_raw[];
    T *ring = (T *)fold_raw;                                                // [NS][R][FD]
    __shared__ __align__(8) uint64_t full[FOLD_NS], empty[FOLD_NS];
    const int nd = (int)*cd.nd;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int k = blockIdx.x * FD + lane;
    // barrier phases run on across the slots this CTA folds: global stage G
    // (counted over all of them) uses buffer G % NS, as its (G / NS)-th fill
    if (tid < FOLD_NS) {
        fbar_init(&full[tid], 1);
        fbar_init(&empty[tid], 1);
    }
    __syncthreads();
    int J0 = 0;
    // grid row 0 folds only the first slot -- the one with the most pending
    // rows (the resolve puts it first), so its long chain starts at once; the
    // other rows share the remaining slots
    const int dstart = blockIdx.y, dstep = blockIdx.y == 0 ? nd : (int)gridDim.y - 1;
    for (int di = dstart; di < nd; di += dstep) {
        const int slot = cd.meta[CD_SLOT * cd.ldm + di];
        const int p0 = cd.off[di], p1 = cd.off[di + 1];
        const int nst = (p1 - p0 + R - 1) / R;
        if (wid == 0) {
            // consumer: the float64 chain, one dimension per lane.  Every row is
            // a plain add: a slot seeded in this batch starts from -0.0 (its
            // seed row then lands exactly: -0 + v = v, like the reference's
            // sum = feature.copy()), skipped rows hold -0.0 (x + -0 = x for
            // every x), so the chain is one dadd per row (~18 cycles on B200).
            const int fp = cd.meta[CD_FP * cd.ldm + di], sp = cd.meta[CD_SP * cd.ldm + di];
            double acc = (sp >= 0 && sp >= fp) ? -0.0 : (k < D ? S[(int64_t)slot * D + k] : 0.0);
            const bool prof = fprof && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0;
            long long tw = 0, tc = 0, t0 = prof ? clock64() : 0;
            for (int j = 0; j < nst; j++) {
                const int G = J0 + j, buf = G % FOLD_NS;
                long long ta = prof ? clock64() : 0;
                fbar_wait(&full[buf], (uint32_t)((G / FOLD_NS) & 1));
                long long tb = prof ? clock64() : 0;
                const int nr = min(R, p1 - p0 - j * R);
                const T *rb = ring + (size_t)buf * R * FD + lane;
#pragma unroll 8
                for (int r = 0; r < nr; r++) acc = dadd(acc, to_d(rb[r * FD]));
                __syncwarp();
                if (lane == 0) fbar_arrive(&empty[buf]);
                if (prof) {
                    tw += tb - ta;
                    tc += clock64() - tb;
                }
            }
            if (prof) {
                atomicAdd((unsigned long long *)&fprof[0], (unsigned long long)tw);
                atomicAdd((unsigned long long *)&fprof[1], (unsigned long long)tc);
                atomicAdd((unsigned long long *)&fprof[2], (unsigned long long)(clock64() - t0));
                atomicAdd((unsigned long long *)&fprof[3], (unsigned long long)(p1 - p0));
                atomicAdd((unsigned long long *)&fprof[4], 1ull);
            }
            if (k < D) {
                S[(int64_t)slot * D + k] = acc;
                if (cd.meta[CD_EV * cd.ldm + di]) {  // sealed at eviction: its final centroid
                    const int cid = cd.meta[CD_CID * cd.ldm + di];
                    fcent[(int64_t)cid * D + k] = ddiv(acc, (double)cd.meta[CD_NFEAT * cd.ldm + di]);
                    if (k == 0) {
                        cl_nfeat[cid] = cd.meta[CD_NFEAT * cd.ldm + di];
                        cl_size[cid] = cd.meta[CD_SIZE * cd.ldm + di];
                    }
                }
            }
        } else {
            // producer for buffer w: global stages G = w (mod NS).  The row
            // pointers of a stage are gathered before its buffer is free
            // (lane l loads rows l, l+32, ...: coalesced, independent), so a
            // refill costs only the copies once the consumer releases it.
            const int w = wid - 1;
            auto gather = [&](int j, const T **rp) {
                const int rbase = p0 + j * R, nr = min(R, p1 - rbase);
#pragma unroll
                for (int c = 0; c < R / 32; c++)
                    rp[c] = (j < nst && c * 32 + lane < nr) ? (const T *)cd.rows[rbase + c * 32 + lane] : nullptr;
            };
            const T *rp[R / 32];
            int j = (w - J0 % FOLD_NS + FOLD_NS) % FOLD_NS;
            gather(j, rp);
            for (; j < nst; j += FOLD_NS) {
                const int G = J0 + j;
                const int nr = min(R, p1 - p0 - j * R);
                if (G >= FOLD_NS) fbar_wait(&empty[w], (uint32_t)(((G / FOLD_NS) - 1) & 1));
                T *dst = ring + (size_t)w * R * FD;
#pragma unroll
                for (int c = 0; c < R / 32; c++) {
                    for (int i = 0; i < 32; i++) {
                        const int row = c * 32 + i;
                        if (row >= nr) break;
                        const T *src = (const T *)__shfl_sync(0xffffffffu, (unsigned long long)rp[c], i);
                        T *d = dst + (size_t)row * FD + lane;
                        if (src != nullptr)
                            cp_async_el((uint32_t)__cvta_generic_to_shared(d), (const void *)(src + k), k < D,
                                        (int)sizeof(T));
                        else
                            *d = (T)(-0.0);  // member already folded by the resolve's exact path
                    }
                }
                gather(j + FOLD_NS, rp);  // next stage's pointers while these copies fly
                asm volatile("cp.async.wait_all;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) fbar_arrive(&full[w]);
            }
        }
        J0 += nst;
    }
    // the last CTA to finish publishes the chain's completion (k_resolve's
    // exact path waits for it)
    __syncthreads();
    if (threadIdx.x == 0 && done_ctas) {
        __threadfence();
        if (atomicAdd(done_ctas, 1u) == gridDim.x * gridDim.y - 1) {
            *done_ctas = 0;
            __threadfence();
            atomicAdd(chain_epoch, 1ull);
        }
    }
}


// finalize: live clusters' final centroids and sizes
__global__ void k_final_live(int D, const int64_t *__restrict__ ctr, const int32_t *__restrict__ live,
                             const double *__restrict__ S, const int32_t *__restrict__ s_nfeat,
                             const int32_t *__restrict__ s_cid, const int32_t *__restrict__ s_size,
                             double *__restrict__ fcent, int32_t *__restrict__ cl_nfeat, int32_t *__restrict__ cl_size) {
    const int i = blockIdx.x;  // live index on x: L can exceed the 65535 limit of grid y
    if (i >= (int)ctr[C_NLIVE]) return;
    const int slot = live[i];
    const int cid = s_cid[slot];
    const double n = (double)s_nfeat[slot];
    for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < D; k += gridDim.y * blockDim.x)
        fcent[(int64_t)cid * D + k] = ddiv(S[(int64_t)slot * D + k], n);
    if (blockIdx.y == 0 && threadIdx.x == 0) {
        cl_nfeat[cid] = s_nfeat[slot];
        cl_size[cid] = s_size[slot];
    }
}

// dups inherit the cluster of the classified object they follow; member rank
// continues that object's rank (ingest.py:69-71, clustering.py:61-63)
__global__ void k_dup_members(int64_t n, const uint8_t *__restrict__ is_dup, const int64_t *__restrict__ anchor_obj,
                              int32_t *__restrict__ cluster_of, int32_t *__restrict__ mrank,
                              int32_t *__restrict__ frank) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || !is_dup[i]) return;
    int64_t a = anchor_obj[i];
    cluster_of[i] = cluster_of[a];
    mrank[i] = mrank[a] + (int32_t)(i - a);
    frank[i] = -1;
}

// anchor (last classified object at or before i) via the classified prefix
__global__ void k_anchor(int64_t n, const uint8_t *__restrict__ is_dup, const int64_t *__restrict__ excl_all,
                         const int64_t *__restrict__ cls_obj, int64_t *__restrict__ anchor) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    anchor[i] = is_dup[i] ? cls_obj[excl_all[i] - 1] : i;
}

// ---------------------------------------------------------------------------
// Deferred seal (clustering.py:71-83): exact float64 distance of every
// featured member to its cluster's final centroid; first minimum wins.
// ---------------------------------------------------------------------------

template <typename T>
__global__ void __launch_bounds__(256) k_seal_dist(int64_t nfeat_total, int D, const int32_t *__restrict__ fmem_cls,
                                                   const int32_t *__restrict__ fmem_cid, const char *const *__restrict__ frow,
                                                   const double *__restrict__ fcent, const PwPlan *__restrict__ plan,
                                                   unsigned long long *__restrict__ best_bits, double *__restrict__ dout) {
    extern __shared__ double sscratch[];
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5;
    const int per = plan->n_chains + plan->n_leaves + plan->n_ops;
    double *scr = sscratch + w * per;
    // each warp takes a contiguous run of members (members are grouped by
    // cluster): the per-cluster minimum is kept in a register and published
    // with one atomic per cluster run, not one per member
    const int64_t nw = (int64_t)gridDim.x * wpb, gw = (int64_t)blockIdx.x * wpb + w;
    const int64_t chunk = (nfeat_total + nw - 1) / nw;
    const int64_t m0 = gw * chunk, m1 = min(nfeat_total, m0 + chunk);
    int cur = -1;
    unsigned long long best = ~0ull;
    for (int64_t m = m0; m < m1; m++) {
        const int cid = fmem_cid[m];
        const T *f = (const T *)frow[fmem_cls[m]];
        const double *c = fcent + (int64_t)cid * D;
        double s = pw_sum_warp(*plan, [&](int k) {
            double x = dsub(c[k], to_d(f[k]));
            return dmul(x, x);
        }, scr);
        double d = __dsqrt_rn(s);
        if ((threadIdx.x & 31) == 0) {
            dout[m] = d;
            if (cid != cur) {
                if (cur >= 0) atomicMin(&best_bits[cur], best);
                cur = cid;
                best = ~0ull;
            }
            best = min(best, (unsigned long long)__double_as_longlong(d));
        }
    }
    if ((threadIdx.x & 31) == 0 && cur >= 0) atomicMin(&best_bits[cur], best);
}

// Screened seal.  k_seal_c32 rounds the final centroids to fp32 (and their
// norms); k_seal_screen measures every featured member against its fp32
// centroid in fp32 (float4 loads, the centroid row L1-resident for a warp's
// run of members), d32, with |d_exact - d32| <= eps1 d32 + eps2:
//   eps1 covers the fp32 terms and sum ((D + 3) 2^-24 relative on the squared
//   sum), eps2 = 2^-24 ||c|| the rounding of the centroid (triangle
//   inequality).  Per cluster U = min (d32 (1 + eps1) + eps2); k_seal_exact
// computes the float64 distance in numpy's pairwise order (the reference's
// np.linalg.norm, clustering.py:77) only for members with
// d32 (1 - eps1) - eps2 <= U -- the minimum and its near-ties -- and leaves
// +inf for the rest, so the pick (first minimum) is unchanged.
__global__ void k_seal_c32(int64_t C, int D, const double *__restrict__ fcent, float *__restrict__ c32,
                           float *__restrict__ cnorm) {
    __shared__ double red[32];
    for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
        double acc = 0.0;
        for (int k = threadIdx.x; k < D; k += blockDim.x) {
            const double v = fcent[c * D + k];
            c32[c * D + k] = (float)v;
            acc += v * v;
        }
        acc = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
            cnorm[c] = (float)(sqrt(t) * (1.0 + 1e-6));
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_seal_screen(int64_t nfeat_total, int D, const int32_t *__restrict__ fmem_cls,
                                                     const int32_t *__restrict__ fmem_cid,
                                                     const char *const *__restrict__ frow,
                                                     const float *__restrict__ c32, const float *__restrict__ cnorm,
                                                     float eps1, float *__restrict__ dlo,
                                                     unsigned int *__restrict__ ubits) {
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * wpb, gw = (int64_t)blockIdx.x * wpb + w;
    const int64_t chunk = (nfeat_total + nw - 1) / nw;
    const int64_t m0 = gw * chunk, m1 = min(nfeat_total, m0 + chunk);
    int cur = -1;
    unsigned int best = ~0u;
    for (int64_t m = m0; m < m1; m++) {
        const int cid = fmem_cid[m];
        const T *f = (const T *)frow[fmem_cls[m]];
        const float *c = c32 + (int64_t)cid * D;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int k = lane;
#pragma unroll 2
        for (; k + 224 < D; k += 256) {
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const float x = __ldg(c + k + 32 * u) - (float)f[k + 32 * u];
                acc[u] = fmaf(x, x, acc[u]);
            }
        }
        for (; k < D; k += 32) {
            const float x = __ldg(c + k) - (float)f[k];
            acc[0] = fmaf(x, x, acc[0]);
        }
        float t = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) {
            const float d = sqrtf(t);
            const float e2 = cnorm[cid] * 5.96046448e-08f * 1.01f;
            dlo[m] = d * (1.f - eps1) - e2;
            const float up = (d * (1.f + eps1) + e2) * (1.f + 1e-6f);
            if (cid != cur) {
                if (cur >= 0) atomicMin(&ubits[cur], best);
                cur = cid;
                best = ~0u;
            }
            best = min(best, __float_as_uint(up));  // non-negative: bit order = value order
        }
    }
    if (lane == 0 && cur >= 0) atomicMin(&ubits[cur], best);
}

template <typename T>
__global__ void __launch_bounds__(256) k_seal_exact(int64_t nfeat_total, int D, const int32_t *__restrict__ fmem_cls,
                                                    const int32_t *__restrict__ fmem_cid,
                                                    const char *const *__restrict__ frow,
                                                    const double *__restrict__ fcent, const PwPlan *__restrict__ plan,
                                                    const float *__restrict__ dlo,
                                                    const unsigned int *__restrict__ ubits,
                                                    unsigned long long *__restrict__ best_bits,
                                                    double *__restrict__ dout) {
    extern __shared__ double sscratch[];
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per = plan->n_chains + plan->n_leaves + plan->n_ops;
    double *scr = sscratch + w * per;
    const int64_t base = ((int64_t)blockIdx.x * wpb + w) * 32;
    if (base >= nfeat_total) return;
    const int64_t m = base + lane;
    bool cand = false;
    int cid = -1;
    if (m < nfeat_total) {
        cid = fmem_cid[m];
        cand = dlo[m] <= __uint_as_float(ubits[cid]);
        if (!cand) dout[m] = __longlong_as_double(0x7ff0000000000000ll);  // +inf: never the minimum
    }
    for (unsigned b = __ballot_sync(0xffffffffu, cand); b; b &= b - 1) {
        const int l = __ffs(b) - 1;
        const int64_t mm = base + l;
        const int cc = __shfl_sync(0xffffffffu, cid, l);
        const T *f = (const T *)frow[fmem_cls[mm]];
        const double *c = fcent + (int64_t)cc * D;
        const double sx = pw_sum_warp(*plan, [&](int k) {
            const double x = dsub(c[k], to_d(f[k]));
            return dmul(x, x);
        }, scr);
        if (lane == 0) {
            const double d = __dsqrt_rn(sx);
            dout[mm] = d;
            atomicMin(&best_bits[cc], (unsigned long long)__double_as_longlong(d));
        }
    }
}

__global__ void k_seal_pick(int64_t nfeat_total, const int32_t *__restrict__ fmem_cid, const int64_t *__restrict__ foff,
                            const double *__restrict__ dout, const unsigned long long *__restrict__ best_bits,
                            int *__restrict__ best_pos) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= nfeat_total) return;
    int cid = fmem_cid[m];
    if ((unsigned long long)__double_as_longlong(dout[m]) == best_bits[cid])
        atomicMin(&best_pos[cid], (int)(m - foff[cid]));
}

// ---------------------------------------------------------------------------
// host-side orchestration
// ---------------------------------------------------------------------------

void launch_screen_tc(int nA, int64_t a0, const char *const *frow, const float *fnorm, int D, const int64_t *nB_dev,
                      int nB_max, const float *C32, const int32_t *snap, const float *cn2, float *out, int64_t ld,
                      cudaStream_t st, float *fnorm_out, ScreenModel sm, double T, int32_t *res_col,
                      int32_t *res_pos, int64_t *nres, int *rowmin_g, float *snorm,
                      const CUtensorMap *tmA, const CUtensorMap *tmB, int rbase, int nR, const int32_t *rmap);
bool make_rows_map(CUtensorMap *tm, const void *base, int64_t rows, int D, int64_t row_bytes, int box_rows);
int64_t scan_i32_to_i64(const int32_t *in, int64_t n, int64_t *out_excl, cudaStream_t st, int64_t *scratch_total);
void scan_u8_to_i64(const uint8_t *in, int64_t n, int invert, int64_t *out_excl, int64_t *d_total, cudaStream_t st);

static double screen_rel(int D) {
    const double u = 5.9604644775390625e-08;  // 2^-24
    double g = (3.0 + 64.0 + (double)((D + 63) / 64) + 2.0) * u;
    return 2.0 * (g / 2.0 + u) + 1e-12;
}

// dynamic shared memory of k_resolve for batch capacity Bc (static smem ~39 KB on top)
size_t resolve_obj_bytes(int Bc, const PwPlan &P) {
    return (size_t)Bc * (9 * 4 + 2 + 1) + 16 + sizeof(double) * (P.n_chains + P.n_leaves + P.n_ops + 8);
}
size_t resolve_smem(int Bc, const PwPlan &P) {
    return (size_t)RS_WCNT_BYTES + (Bc > 4096 ? 16 : resolve_obj_bytes(Bc, P));
}

// FP32 snapshot packed in snapshot order (TMA boxes of the TC screen need
// consecutive rows): C32q[q] = C32[snap[q]], q < nsnap.
__global__ void k_snap_pack(const int64_t *__restrict__ ctr, const int32_t *__restrict__ snap,
                            const float *__restrict__ C32, float *__restrict__ C32q, int D) {
    pdl_enter();
    const int nsnap = (int)ctr[C_NSNAP];
    const int n4 = D >> 2;
    for (int q = blockIdx.x; q < nsnap; q += gridDim.x) {
        const float4 *src = (const float4 *)(C32 + (int64_t)snap[q] * D);
        float4 *dst = (float4 *)(C32q + (int64_t)q * D);
        for (int k = threadIdx.x; k < n4; k += blockDim.x) dst[k] = src[k];
    }
}

// object rows (relative to the ingest call's feature rows) of the first and
// last classified object of each batch
__global__ void k_batch_rows(int nb, const int64_t *__restrict__ cfirst, const int64_t *__restrict__ clast,
                             const int64_t *__restrict__ cls_obj, int64_t obj0, int64_t *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb) return;
    out[2 * i] = cls_obj[cfirst[i]] - obj0;
    out[2 * i + 1] = cls_obj[clast[i]] - obj0;
}

template <typename T>
void run_batches(fx_stream *s, int64_t c_begin, int64_t c_end) {
    cudaStream_t st = s->st;
    // batches are capped at 1/age_div of the objects seen so far (young clusters stay decidable)
    static const int64_t age_div = getenv("FOCUS_B200_AGE_DIV") ? std::max(1, atoi(getenv("FOCUS_B200_AGE_DIV"))) : 4;
    // Several engines ingesting on one device: programmatic dependent launch
    // parks each dependent grid's CTAs on SMs before its primary finishes, and
    // with many engines those parked CTAs starve other engines' large-shared-
    // memory CTAs (the TC screen, the resolve) for up to seconds (CUPTI traces,
    // DESIGN.md §6).  So with more than one live engine: no PDL, and the
    // exact chain on the main stream.
    const bool multi_inline = live_engines(s->dev, 0) > 1 && !s->partitioned;
    struct PdlScope {
        explicit PdlScope(bool on) { pdl_suppress(on); }
        ~PdlScope() { pdl_suppress(false); }
    } pdl_scope_(multi_inline);
    const int D = s->cfg.dim;
    const float rel = (float)screen_rel(D);
    const float absc = (float)(2.0 * 2.384185791015625e-07);  // 2^-22 * 2
    // TF32 dot error gamma = 2^-9 + D 2^-22 (operand rounding + FP32 accumulation), d^2 error 2 gamma |a||b|
    const double gam = 1.953125e-03 + (double)D * 2.384185791015625e-07;
    const ScreenModel sm{s->tc_screen ? 1 : 0, rel, absc, (float)(2.0 * gam * 1.01), (float)(256.0 * 5.9604644775390625e-08)};
    // TMA operand staging for the TC screen (fp32 rows, 16-byte aligned): A
    // boxes over the ingest call's feature rows, B boxes over the packed snapshot
    CUtensorMap tmA, tmB;
    static const bool tma_off = getenv("FOCUS_B200_TCLOAD") && std::string(getenv("FOCUS_B200_TCLOAD")) == "cp";
    bool tma = s->tc_screen && sizeof(T) == 4 && !tma_off && s->abase && s->rows_aligned16 && D % 4 == 0;
    if (tma) {
        s->C32q.reserve((size_t)s->ld * D);
        tma = make_rows_map(&tmA, s->abase, s->arows, D, (int64_t)D * 4, 128) &&
              make_rows_map(&tmB, s->C32q.p, s->ld, D, (int64_t)D * 4, 128);
    }
    // batch boundaries (as the loop below forms them) and, for features with
    // duplicate rows, each batch's span of object rows (one readback per call)
    std::vector<int64_t> bfirst, blast, brows;
    if (tma) {
        for (int64_t c0 = c_begin, B = 0; c0 < c_end; c0 += B) {
            const int64_t cap = std::max<int64_t>(64, (std::max<int64_t>(c0, 0) / age_div / 64) * 64);
            B = std::min<int64_t>(std::min<int64_t>(s->B, cap), c_end - c0);
            bfirst.push_back(c0);
            blast.push_back(c0 + B - 1);
        }
        const int nb = (int)bfirst.size();
        brows.resize(2 * (size_t)nb);
        if (s->a_compact) {
            for (int i = 0; i < nb; i++) {
                brows[2 * i] = bfirst[i] - s->a_cbase;
                brows[2 * i + 1] = blast[i] - s->a_cbase;
            }
        } else if (nb > 0) {
            DevBuf<int64_t> d_in, d_out;
            d_in.reserve(2 * (size_t)nb);
            d_out.reserve(2 * (size_t)nb);
            FX_CUDA(cudaMemcpyAsync(d_in.p, bfirst.data(), sizeof(int64_t) * nb, cudaMemcpyHostToDevice, st));
            FX_CUDA(cudaMemcpyAsync(d_in.p + nb, blast.data(), sizeof(int64_t) * nb, cudaMemcpyHostToDevice, st));
            k_batch_rows<<<(unsigned)cdiv(nb, 256), 256, 0, st>>>(nb, d_in.p, d_in.p + nb, s->cls_obj.p, s->a_obj0,
                                                                 d_out.p);
            FX_LAUNCHED();
            FX_CUDA(cudaMemcpyAsync(brows.data(), d_out.p, sizeof(int64_t) * 2 * nb, cudaMemcpyDeviceToHost, st));
            FX_CUDA(cudaStreamSynchronize(st));
        }
    }
    int bi = 0;
    using hclock = std::chrono::steady_clock;
    auto hms = [](hclock::time_point a, hclock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::vector<double> chk_expect;
    std::vector<int32_t> chk_slots;
    // fused row pass: FP32 rows, D % 4 == 0, D <= 2048, 16-byte aligned rows
    const bool rowpass = sizeof(T) == 4 && D % 4 == 0 && D <= 2048 && s->rows_aligned16;
    // large snapshots (C3): one CTA per object scans its distance row (k_rowpass_wide)
    static const int wide_min = getenv("FOCUS_B200_RP_WIDE") ? atoi(getenv("FOCUS_B200_RP_WIDE")) : 4096;
    const bool use_wide = rowpass && wide_min > 0 && s->ld > wide_min && D > 1024;
    for (int64_t c0 = c_begin, B = 0; c0 < c_end; c0 += B, bi++) {
        const auto h0 = hclock::now();
        const int cbuf = (int)(s->batch_no & 1);  // chain descriptor buffer of this batch
        // the drift bound grows like (batch size / objects so far): keep batches
        // at <= 1/4 of the stream's age so young clusters stay decidable by bounds
        const int64_t age = std::max<int64_t>(c0, 0);
        const int64_t cap = std::max<int64_t>(64, (age / age_div / 64) * 64);
        B = (int)std::min<int64_t>(std::min<int64_t>(s->B, cap), c_end - c0);
        s->t_ms[6] += 1.0;
        // 1. snapshot screen
        bool fused_res = false;
        s->tstart(1);
        if (s->tc_screen) {
            // the screen also produces ||f|| of the batch rows (fnorm) unless an earlier pass did
            // fused: residual detection when the snapshot fits one column tile
            fused_res = s->ld <= 128;
            int rbase = 0, nR = B;
            if (tma) {
                rbase = (int)brows[2 * bi];
                nR = (int)(brows[2 * bi + 1] - brows[2 * bi] + 1);
                launch_pdl(k_snap_pack, dim3((unsigned)std::min<int64_t>(s->ld, 148 * 4)), dim3(128), 0, st, s->ctr.p, s->snap_slot.p,
                                                                                        s->C32.p, s->C32q.p, D);
                FX_LAUNCHED();
            }
            launch_screen_tc(B, c0, s->frow.p, s->fnorm.p, D, s->ctr.p + C_NSNAP, (int)s->ld, s->C32.p,
                             s->snap_slot.p, s->s_cn2.p, s->dist.p, s->ld, st, s->has_fc ? nullptr : s->fnorm.p, sm,
                             s->cfg.t, fused_res ? s->res_col.p : nullptr, s->res_pos.p, s->ctr.p + C_NRES,
                             s->rowmin.p, s->snorm.p, tma ? &tmA : nullptr, tma ? &tmB : nullptr, rbase, nR,
                             s->a_compact ? nullptr : s->orow.p);
        } else {
            const unsigned grid = (unsigned)std::min<int64_t>(cdiv(s->ld, SC_T) * cdiv(B, SC_T), 148 * 8);
            FromSnapshot fb{s->C32.p, s->snap_slot.p, D};
            k_screen<T, FromSnapshot><<<grid, 256, 0, st>>>(B, c0, s->frow.p, D, s->ctr.p + C_NSNAP, (int)s->ld, fb,
                                                            s->dist.p, s->ld);
            FX_LAUNCHED();
        }
        s->tstop();
        s->tstart(7);  // residual detection + columns
        // 2. residuals + their in-batch columns
        {
            if (!fused_res && s->tc_screen) {
                launch_pdl(k_res_from_min, dim3((unsigned)cdiv(B, 256)), dim3(256), 0, st, B, s->rowmin.p, s->cfg.t, s->res_col.p,
                                                                      s->res_pos.p, s->ctr.p + C_NRES);
                FX_LAUNCHED();
            } else if (!fused_res) {
                launch_pdl(k_residuals, dim3((unsigned)cdiv((int64_t)B * 32, 256)), dim3(256), 0, st, 
                    B, s->ctr.p, s->dist.p, s->ld, s->s_cn2.p, s->snap_slot.p, s->fnorm.p, c0, sm, s->cfg.t,
                    s->res_col.p, s->res_pos.p, s->ctr.p + C_NRES);
                FX_LAUNCHED();
            }
            const bool rc_ok = D <= 6144 && !use_wide;  // RC_COLS staged rows fit in shared memory; the wide
                                                        // row pass leaves every residual column to the tiled kernel
            if (rc_ok && !rowpass) {
                const size_t smem = sizeof(float) * RC_COLS * D;
                static size_t rc_set[64] = {};
                size_t &cur = rc_set[dev_slot()];
                if (smem > 48 * 1024 && smem > cur) {
                    FX_CUDA(cudaFuncSetAttribute(k_res_cols<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    cur = smem;
                }
                k_res_cols<T><<<148, 256, smem, st>>>(B, c0, s->frow.p, D, s->ctr.p + C_NRES, s->res_pos.p, s->dres.p, B);
                FX_LAUNCHED();
            }
            const unsigned grid = (unsigned)std::min<int64_t>(cdiv(B, SC_T) * cdiv(B, SC_T), 148);
            FromResidual<T> fb{s->frow.p, c0, s->res_pos.p};
            launch_pdl(k_screen<T, FromResidual<T>>, dim3(grid), dim3(256), 0, st, B, c0, s->frow.p, D, s->ctr.p + C_NRES, B, fb, s->dres.p, B,
                                                               rc_ok ? RC_MAX : -1);
            FX_LAUNCHED();
        }
        s->tstop();
        s->tstart(15);  // row summary (+ fp32 refine of the best candidate)
        const float *snorm = s->tc_screen ? s->snorm.p : nullptr;
        if (rowpass) {
            const unsigned grid = (unsigned)std::min<int64_t>(cdiv((int64_t)B * 32, 256), 148 * 8);
            static const int rp_minb = getenv("FOCUS_B200_RP_MINB") ? atoi(getenv("FOCUS_B200_RP_MINB")) : 2;
            static const bool rp_lean = !(getenv("FOCUS_B200_RP_LEAN") && atoi(getenv("FOCUS_B200_RP_LEAN")) == 0);
            if (use_wide)
                launch_pdl(k_rowpass_wide, dim3((unsigned)std::min<int64_t>(B, 148 * 8)), dim3(RPW_T), 0, st, B, c0,
                           s->frow.p, D, s->ctr.p, s->dist.p, s->ld, s->s_cn2.p, s->snap_slot.p, s->fnorm.p, sm, rel,
                           absc, s->C32.p, s->sum_slot.p, s->sum_q.p, s->sum_d1.p, s->sum_e1.p, s->sum_lbr.p, snorm);
            else if (rp_lean && D > 1024)
                launch_pdl(k_rowpass_lean, dim3((unsigned)std::min<int64_t>(cdiv((int64_t)B * 32, 256), 148 * 4)),
                           dim3(256), 0, st, B, c0, s->frow.p, D, s->ctr.p, s->dist.p, s->ld, s->s_cn2.p,
                           s->snap_slot.p, s->fnorm.p, sm, rel, absc, s->C32.p, s->cfg.t, s->res_pos.p, s->dres.p, B,
                           s->sum_slot.p, s->sum_q.p, s->sum_d1.p, s->sum_e1.p, s->sum_lbr.p, snorm);
            else if (D <= 1024)
                launch_pdl(k_rowpass<8, 2>, dim3(grid), dim3(256), 0, st, B, c0, s->frow.p, D, s->ctr.p, s->dist.p, s->ld, s->s_cn2.p,
                                                   s->snap_slot.p, s->fnorm.p, sm, rel, absc, s->C32.p, s->cfg.t,
                                                   s->res_pos.p, s->dres.p, B, s->sum_slot.p, s->sum_q.p, s->sum_d1.p,
                                                   s->sum_e1.p, s->sum_lbr.p, snorm);
            else
                launch_pdl(rp_minb >= 3 ? k_rowpass<16, 3> : k_rowpass<16, 2>, dim3(grid), dim3(256), 0, st, B, c0, s->frow.p, D, s->ctr.p, s->dist.p, s->ld, s->s_cn2.p,
                                                    s->snap_slot.p, s->fnorm.p, sm, rel, absc, s->C32.p, s->cfg.t,
                                                    s->res_pos.p, s->dres.p, B, s->sum_slot.p, s->sum_q.p, s->sum_d1.p,
                                                   s->sum_e1.p, s->sum_lbr.p, snorm);
            FX_LAUNCHED();
        } else {
        launch_pdl(k_row_summary<T>, dim3((unsigned)cdiv((int64_t)B * 32, 256)), dim3(256), 0, st, 
                B, s->ctr.p, s->dist.p, s->ld, s->s_cn2.p, s->snap_slot.p, s->fnorm.p, c0, sm, rel, absc, s->frow.p,
                s->C32.p, D, s->sum_slot.p, s->sum_q.p, s->sum_d1.p, s->sum_e1.p, s->sum_lbr.p, snorm);
            FX_LAUNCHED();
        }
        s->tstop();
        const auto h1 = hclock::now();
        s->t_ms[8] += hms(h0, h1);
        // 3. resolve (parallel verified segments + exact sequential events)
        s->tstart(2);
        {
            ResolveArgs A;
            A.B = B;
            A.Bcap = s->B;
            A.c0 = c0;
            A.D = D;
            A.T = s->cfg.t;
            A.M = s->cfg.m;
            A.rel = rel;
            A.absc = absc;
            A.sm = sm;
            A.dist = s->dist.p;
            A.ld = s->ld;
            A.dres = s->dres.p;
            A.ldr = B;
            A.res_col = s->res_col.p;
            A.res_pos = s->res_pos.p;
            A.dod = s->dod.p;
            A.frow = s->frow.p;
            A.fnorm = s->fnorm.p;
            A.dup_run = s->dup_run.p;
            A.cls_obj = s->cls_obj.p;
            A.S = s->S.p;
            A.s_cid = s->s_cid.p;
            A.s_nfeat = s->s_nfeat.p;
            A.s_size = s->s_size.p;
            A.s_snapq = s->s_snapq.p;
            A.s_seedpos = s->s_seedpos.p;
            A.s_foldpos = s->s_foldpos.p;
            A.s_pend = s->s_pend.p;
            A.s_odcol = s->s_odcol.p;
            A.s_evicted = s->s_evicted.p;
            A.s_didx = s->s_didx.p;
            A.s_drift = s->s_drift.p;
            A.s_cn2 = s->s_cn2.p;
            A.live = s->live.p;
            A.live_pos = s->live_pos.p;
            A.free_stack = s->free_stack.p;
            A.defer_free = s->defer_free.p;
            A.snap_slot = s->snap_slot.p;
            A.ctr = s->ctr.p;
            A.slot_of = s->slot_of.p;
            A.pend_rank = s->pend_rank.p;
            A.evict_slot = s->evict_slot.p;
            A.evict_cid = s->evict_cid.p;
            A.cid_slot = s->cid_slot.p;
            A.s_fjoin = s->s_fjoin.p;
            A.ev_pos = s->ev_pos.p;
            A.ev_vic = s->ev_vic.p;
            A.dirty = s->dirty.p;
            A.dirty_off = s->dirty_off.p;
            A.pend_list = s->pend_list.p;
            A.pend_seg = s->pend_seg.p;
            A.cluster_of = s->cluster_of.p;
            A.mrank = s->mrank.p;
            A.frank = s->frank.p;
            A.plan = s->plan.p;
            A.s_grp = s->s_grp.p;
            A.prof = (long long *)s->prof.p;
            A.batch_no = (int)s->batch_no;
            A.sum_slot = s->sum_slot.p;
            A.sum_q = s->sum_q.p;
            A.sum_d1 = s->sum_d1.p;
            A.sum_e1 = s->sum_e1.p;
            A.sum_lbr = s->sum_lbr.p;
            A.h_ring = s->h_ctr_ring + (s->batch_no % 3) * C_COUNT;
            A.f_rank = s->f_rank.p;
            A.f_dup = s->f_dup.p;
            A.f_P = s->f_P.p;
            A.f_ccnt = s->f_ccnt.p;
            A.f_cdup = s->f_cdup.p;
            A.f_csum = s->f_csum.p;
            A.f_cmax = s->f_cmax.p;
            A.f_gi = s->f_gi.p;
            A.f_gf = s->f_gf.p;
            A.f_gd = s->f_gd.p;
            A.s_sdev = s->s_sdev.p;
            A.rs_gobj = s->B > 4096 ? s->rs_gobj.p : nullptr;
            // fast path first (the common all-certain batch over the whole
            // grid); k_resolve returns at once when it committed
            static const bool nofast = getenv("FOCUS_B200_NOFAST") && atoi(getenv("FOCUS_B200_NOFAST"));
            const PwPlan &P = *s->plan_host;
            size_t smem = resolve_smem(s->B, P);
            auto kern = k_resolve<T>;
            static size_t smem_set[64] = {};
            size_t &cur = smem_set[dev_slot()];
            if (smem > cur) {
                FX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                cur = smem;
            }
            // fast path first (the common all-certain batch over the whole
            // grid); k_resolve returns at once when it committed
            if (!nofast) {
                const unsigned nch = (unsigned)cdiv(B, RF_T);
                launch_pdl(k_rfast1, dim3(nch), dim3(RF_T), 0, st, A);
                FX_LAUNCHED();
                launch_pdl(k_rfast3, dim3(nch), dim3(RF_T), 0, st, A);
                FX_LAUNCHED();
            }
            // its exact path reads the reference's float64 sums: the previous
            // batch's chain must be done -- the resolve waits for it on the
            // device, and only when it takes the exact path (inline chains are
            // stream-ordered already)
            if (multi_inline || !s->chain_epoch.p) {
                if (s->chain_pending[cbuf ^ 1]) FX_CUDA(cudaStreamWaitEvent(st, s->ev_ch[cbuf ^ 1], 0));
                A.chain_epoch = nullptr;
            } else {
                A.chain_epoch = s->chain_epoch.p;
            }
            launch_pdl(kern, dim3(1), dim3(RS_THREADS), smem, st, A);
            FX_LAUNCHED();
        }
        s->tstop();
        const auto h2 = hclock::now();
        s->t_ms[9] += hms(h1, h2);
        // 4. cluster-array capacity for final centroids of evicted clusters,
        //    without a per-batch host sync: each batch creates <= B clusters, so
        //    the count read back (asynchronously) two batches ago + 3B bounds it.
        {
            const int slot_k = (int)(s->batch_no % 3);  // written by the resolve itself (A.h_ring)
            FX_CUDA(cudaEventRecord(s->ring_ev[slot_k], st));
            int64_t known = 0;
            if (s->batch_no >= 2) {
                const int slot_old = (int)((s->batch_no - 2) % 3);
                static const double stall_ms = getenv("FOCUS_B200_STALL") ? atof(getenv("FOCUS_B200_STALL")) : 0.0;
                const auto w0 = hclock::now();
                FX_CUDA(cudaEventSynchronize(s->ring_ev[slot_old]));
                if (stall_ms > 0.0) {
                    const double w = hms(w0, hclock::now()), lb = hms(h0, w0);
                    if (w > stall_ms || lb > stall_ms)
                        fprintf(stderr, "STALL engine %p batch %ld: ring sync %.1f ms, launches before it %.1f ms\n",
                                (void *)s, (long)s->batch_no, w, lb);
                }
                known = s->h_ctr_ring[slot_old * C_COUNT + C_NEXT_CID];
            }
            s->batch_no++;
            const int64_t need = known + 3 * (int64_t)s->B;
            if (need > s->cl_cap) {
                FX_CUDA(cudaStreamSynchronize(st));
                FX_CUDA(cudaStreamSynchronize(s->st2));  // the chain writes fcent / cl_nfeat / cl_size
                int64_t cap = std::max<int64_t>(need, s->cl_cap * 2);
                s->fcent.grow((size_t)cap * D, (size_t)s->cl_cap * D, st);
                s->cl_nfeat.grow(cap, s->cl_cap, st);
                s->cl_size.grow(cap, s->cl_cap, st);
                s->cl_cap = cap;
            }
            if (need > (int64_t)s->cid_slot.n) s->cid_slot.grow((size_t)need, s->cid_slot.n, st);
        }
        const auto h3 = hclock::now();
        s->t_ms[10] += hms(h2, h3);
        if (s->debug_check) {  // FOCUS_B200_CHECK=1: host-side invariants of the resolve output
            FX_CUDA(cudaStreamSynchronize(st));
            FX_CUDA(cudaStreamSynchronize(s->st2));
            int64_t hc[C_COUNT];
            FX_CUDA(cudaMemcpy(hc, s->ctr.p, sizeof(hc), cudaMemcpyDeviceToHost));
            const int nd = (int)hc[C_NDIRTY];
            std::vector<int32_t> dr(nd), doff(nd + 1), pl(B), so(B), seedp(s->nslots), foldp(s->nslots);
            FX_CUDA(cudaMemcpy(dr.data(), s->dirty.p, 4 * nd, cudaMemcpyDeviceToHost));
            FX_CUDA(cudaMemcpy(doff.data(), s->dirty_off.p, 4 * (nd + 1), cudaMemcpyDeviceToHost));
            FX_CUDA(cudaMemcpy(pl.data(), s->pend_list.p, 4 * B, cudaMemcpyDeviceToHost));
            FX_CUDA(cudaMemcpy(so.data(), s->slot_of.p, 4 * B, cudaMemcpyDeviceToHost));
            FX_CUDA(cudaMemcpy(seedp.data(), s->s_seedpos.p, 4 * s->nslots, cudaMemcpyDeviceToHost));
            FX_CUDA(cudaMemcpy(foldp.data(), s->s_foldpos.p, 4 * s->nslots, cudaMemcpyDeviceToHost));
            std::vector<int> seen(s->nslots, 0);
            for (int i = 0; i < nd; i++) {
                const int sl = dr[i];
                if (seen[sl]++) fprintf(stderr, "CHECK batch %ld: slot %d dirty twice\n", (long)s->batch_no, sl);
                for (int p = doff[i]; p < doff[i + 1]; p++) {
                    const int b = pl[p];
                    if (b < 0 || b >= B || so[b] != sl || (p > doff[i] && b <= pl[p - 1]))
                        fprintf(stderr, "CHECK batch %ld: slot %d row %d -> pos %d (slot_of %d)\n", (long)s->batch_no, sl,
                                p - doff[i], b, (b >= 0 && b < B) ? so[b] : -9);
                }
                if (seedp[sl] >= 0 && doff[i + 1] > doff[i] && seedp[sl] >= foldp[sl] && pl[doff[i]] != seedp[sl])
                    fprintf(stderr, "CHECK batch %ld: seed slot %d first row %d != seed %d\n", (long)s->batch_no, sl,
                            pl[doff[i]], seedp[sl]);
            }
            if (doff[nd] != B) fprintf(stderr, "CHECK batch %ld: %d pending rows for %ld objects\n", (long)s->batch_no, doff[nd], (long)B);
            if (s->batch_no < 3) fprintf(stderr, "CHECK batch %ld: %d dirty slots ok\n", (long)s->batch_no, nd);
            // expected sums of the dirty slots after the fold (host, sequential float64)
            std::vector<const char *> fr(B);
            FX_CUDA(cudaMemcpy(fr.data(), s->frow.p + c0, sizeof(void *) * B, cudaMemcpyDeviceToHost));
            chk_expect.assign((size_t)nd * D, 0.0);
            chk_slots = dr;
            std::vector<double> srow(D);
            std::vector<T> frw(D);
            for (int i = 0; i < nd; i++) {
                const int sl = dr[i];
                FX_CUDA(cudaMemcpy(srow.data(), s->S.p + (size_t)sl * D, 8 * D, cudaMemcpyDeviceToHost));
                bool fresh = seedp[sl] >= 0 && seedp[sl] >= foldp[sl];
                for (int p = doff[i]; p < doff[i + 1]; p++) {
                    const int b = pl[p];
                    if (b < foldp[sl]) continue;
                    FX_CUDA(cudaMemcpy(frw.data(), fr[b], sizeof(T) * D, cudaMemcpyDeviceToHost));
                    for (int k = 0; k < D; k++) srow[k] = fresh ? (double)frw[k] : srow[k] + (double)frw[k];
                    fresh = false;
                }
                std::copy(srow.begin(), srow.end(), chk_expect.begin() + (size_t)i * D);
            }
        }
        // 5. snapshot tree fold (main stream) + the exact chain one batch behind (st2)
        {
            s->tstart(3);
            const int buf = cbuf;
            // the chain of two batches ago read this buffer's descriptor
            if (s->chain_pending[buf]) FX_CUDA(cudaStreamWaitEvent(st, s->ev_ch[buf], 0));
            const int64_t gxt = cdiv(D, TF_C);
            const int64_t gyt = TF_SPLIT + std::max<int64_t>(4, std::min<int64_t>(2 * (int64_t)B + 1, (148 * 4) / gxt));
            const int ldm = 2 * s->B + 3;
            int32_t *meta = s->cd_meta.p + (size_t)buf * CD_NMETA * ldm;
            int32_t *coff = s->cd_off.p + (size_t)buf * ldm;
            const char **crows = s->cd_rows.p + (size_t)buf * s->B;
            static const bool tf_old = getenv("FOCUS_B200_TFOLD_OLD") && atoi(getenv("FOCUS_B200_TFOLD_OLD"));
            if (tf_old) {
                launch_pdl(k_tfold<T>, dim3((unsigned)gxt, (unsigned)gyt), dim3(TF_T), 0, st, D, c0, B, s->ctr.p,
                           s->dirty.p, s->dirty_off.p, s->pend_list.p, s->frow.p, s->fnorm.p, s->s_nfeat.p,
                           s->s_foldpos.p, s->s_seedpos.p, s->s_evicted.p, s->s_cid.p, s->s_size.p, s->S_tree.p,
                           s->C32.p, s->s_cn2.p, s->s_abs.p, s->s_sdev.p, s->tf_cn2.p, s->tf_cnt.p, s->tf_part.p,
                           s->tf_bcnt.p, s->cd_nd.p + buf, meta, ldm, coff, crows);
            } else {
                const unsigned gx3 = (unsigned)cdiv(D, TF3_T);
                static const bool tf4_off = getenv("FOCUS_B200_TF4") && atoi(getenv("FOCUS_B200_TF4")) == 0;
                static const int tfb_gy = getenv("FOCUS_B200_TFB_GY") ? atoi(getenv("FOCUS_B200_TFB_GY")) : 0;
                if (sizeof(T) == 4 && s->rows_aligned16 && D % 4 == 0 && !tf4_off)
                    launch_pdl(k_tfold_a4, dim3(gx3, (unsigned)cdiv(B, TF3_R)), dim3(TF4_T), 0, st, D, c0, (int)B,
                               s->dirty.p, s->pend_list.p, s->pend_seg.p, s->frow.p, s->fnorm.p, s->s_foldpos.p,
                               s->tf_P.p, s->tf_PF.p, crows);
                else
                    launch_pdl(k_tfold_a<T>, dim3(gx3, (unsigned)cdiv(B, TF3_R)), dim3(TF3_T), 0, st, D, c0, (int)B,
                               s->dirty.p, s->pend_list.p, s->pend_seg.p, s->frow.p, s->fnorm.p, s->s_foldpos.p,
                               s->tf_P.p, s->tf_PF.p, crows);
                FX_LAUNCHED();
                launch_pdl(k_tfold_b, dim3(gx3, (unsigned)std::min<int64_t>(2 * (int64_t)B + 3, tfb_gy > 0 ? tfb_gy : std::max<int64_t>(64, 1184 / gx3))), dim3(TF3_T), 0, st, D, s->ctr.p, s->dirty.p,
                           s->dirty_off.p, s->s_nfeat.p, s->s_foldpos.p, s->s_seedpos.p, s->s_evicted.p, s->s_cid.p,
                           s->s_size.p, s->tf_P.p, s->tf_PF.p, s->S_tree.p, s->C32.p, s->s_cn2.p, s->s_abs.p,
                           s->s_sdev.p, s->tf_cn2.p, s->tf_cnt.p, s->cd_nd.p + buf, meta, ldm, coff);
            }
            FX_LAUNCHED();
            s->tstop();
            // several engines on the device (multi_inline): the chain runs on the
            // main stream -- no cross-stream events; FOCUS_B200_FOLD_INLINE=1 forces it
            static const bool fold_inline_env = getenv("FOCUS_B200_FOLD_INLINE") && atoi(getenv("FOCUS_B200_FOLD_INLINE"));
            const bool fold_inline = fold_inline_env || multi_inline;
            cudaStream_t fst = fold_inline ? st : s->st2;
            if (!fold_inline) {
                FX_CUDA(cudaEventRecord(s->ev_tf[buf], st));
                FX_CUDA(cudaStreamWaitEvent(s->st2, s->ev_tf[buf], 0));
            }
            const int64_t gx = cdiv(D, FD);
            // 4 grid rows (the largest slot on row 0, the rest shared by rows 1-3):
            // the chain is off the critical path, so it is kept narrow (r02aq:
            // 44.1 M objects/s vs 42.8 M with one row per 2B+1 / 27 slots)
            static const int fold_gy = getenv("FOCUS_B200_FOLD_GY") ? atoi(getenv("FOCUS_B200_FOLD_GY")) : 4;
            const int64_t gy = fold_gy > 0 ? std::min<int64_t>(fold_gy, 2 * (int64_t)B + 1)
                                           : std::max<int64_t>(8, std::min<int64_t>(2 * (int64_t)B + 1, (148 * 12) / gx));
            static bool fold_attr[64] = {};
            if (!fold_attr[dev_slot()]) {
                FX_CUDA(cudaFuncSetAttribute(k_fold<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fold_smem<T>()));
                fold_attr[dev_slot()] = true;
            }
            ChainDesc cd{s->cd_nd.p + buf, meta, ldm, coff, crows};
            k_fold<T><<<dim3((unsigned)gx, (unsigned)gy), FOLD_THREADS, fold_smem<T>(), fst>>>(
                D, cd, s->S.p, s->fcent.p, s->cl_nfeat.p, s->cl_size.p, (long long *)(s->prof.p + 16),
                s->fold_done.p, s->chain_epoch.p);  // inline chains count too (the mode can change mid-stream)
            FX_LAUNCHED();
            if (!fold_inline) {
                FX_CUDA(cudaEventRecord(s->ev_ch[buf], s->st2));
                s->chain_pending[buf] = true;
            }
        }
        if (s->debug_check) {
            FX_CUDA(cudaStreamSynchronize(st));
            FX_CUDA(cudaStreamSynchronize(s->st2));
            std::vector<double> srow(D);
            int nbad = 0;
            for (size_t i = 0; i < chk_slots.size(); i++) {
                FX_CUDA(cudaMemcpy(srow.data(), s->S.p + (size_t)chk_slots[i] * D, 8 * D, cudaMemcpyDeviceToHost));
                for (int k = 0; k < D; k++)
                    if (memcmp(&srow[k], &chk_expect[i * D + k], 8) != 0) {
                        if (nbad++ < 5)
                            fprintf(stderr, "CHECK batch %ld: fold slot %d dim %d got %.17g want %.17g\n",
                                    (long)s->batch_no, chk_slots[i], k, srow[k], chk_expect[i * D + k]);
                        break;
                    }
            }
        }
        s->t_ms[11] += hms(h3, hclock::now());
    }
}

template void run_batches<float>(fx_stream *, int64_t, int64_t);
template void run_batches<double>(fx_stream *, int64_t, int64_t);

void launch_dup_flags(fx_stream *s, int64_t n, const int64_t *d_fid, const double *d_sig, uint8_t *d_out) {
    const int S = s->cfg.sig_dim;
    k_dup_flags<<<(unsigned)cdiv(n, DUP_T), DUP_T, 0, s->st>>>(n, S, d_fid, d_sig, s->has_prev ? 1 : 0, s->prev_fid,
                                                           s->prev_sig.p, s->cfg.pixel_eps, d_out);
    FX_LAUNCHED();
}

void launch_dup_flags_raw(int64_t n, int S, const int64_t *d_fid, const double *d_sig, double eps, uint8_t *d_out,
                          cudaStream_t st) {
    k_dup_flags<<<(unsigned)cdiv(n, DUP_T), DUP_T, 0, st>>>(n, S, d_fid, d_sig, 0, 0, nullptr, eps, d_out);
    FX_LAUNCHED();
}

void launch_compact(fx_stream *s, int64_t n, int64_t obj_base, int64_t cls_base, const uint8_t *d_dup,
                    const int64_t *d_excl, const char *feat_base, int compact) {
    const int64_t row_bytes = (int64_t)s->cfg.dim * s->esize;
    s->orow.grow(n, 0, s->st);
    k_compact_cls<<<(unsigned)cdiv(n, 256), 256, 0, s->st>>>(n, obj_base, cls_base, d_dup, d_excl, feat_base,
                                                             row_bytes, compact, s->cls_obj.p, s->frow.p, s->dup_run.p,
                                                             compact ? nullptr : s->orow.p);
    s->abase = feat_base;
    s->a_compact = compact != 0;
    s->a_cbase = cls_base;
    s->a_obj0 = obj_base;
    FX_LAUNCHED();
    k_dup_runs<<<(unsigned)cdiv(n, 256), 256, 0, s->st>>>(n, cls_base, d_dup, d_excl, s->dup_run.p);
    FX_LAUNCHED();
}

void launch_fnorm(fx_stream *s, int64_t c0, int64_t nc) {
    if (nc <= 0) return;
    unsigned grid = (unsigned)cdiv(nc * 32, 256);
    if (s->cfg.feat_type == FX_F64)
        k_fnorm<double><<<grid, 256, 0, s->st>>>(c0, nc, s->cfg.dim, s->frow.p, s->fnorm.p);
    else
        k_fnorm<float><<<grid, 256, 0, s->st>>>(c0, nc, s->cfg.dim, s->frow.p, s->fnorm.p);
    FX_LAUNCHED();
}

void launch_rank(fx_stream *s, int64_t c0, int64_t nc, const int32_t *d_tcls, unsigned long long *d_err) {
    if (nc <= 0) return;
    k_rank_topk<<<(unsigned)cdiv(nc, 256), 256, 0, s->st>>>(c0, nc, s->cls_obj.p, s->oid.p, d_tcls, s->cfg.k,
                                                           s->cfg.vocab, s->gt, s->seed, s->rm_thr.p, s->rm_emit.p,
                                                           s->rm_fill.p, s->topk.p, d_err);
    FX_LAUNCHED();
}

void launch_final_live(fx_stream *s) {
    const int D = s->cfg.dim;
    int64_t L = s->h_ctr[C_NLIVE];
    if (L <= 0) return;
    dim3 grid((unsigned)L, (unsigned)cdiv(D, 256));
    k_final_live<<<grid, 256, 0, s->st>>>(D, s->ctr.p, s->live.p, s->S.p, s->s_nfeat.p, s->s_cid.p, s->s_size.p,
                                          s->fcent.p, s->cl_nfeat.p, s->cl_size.p);
    FX_LAUNCHED();
}

void launch_dup_members(fx_stream *s, int64_t n, const int64_t *d_excl_all, int64_t *d_anchor) {
    k_anchor<<<(unsigned)cdiv(n, 256), 256, 0, s->st>>>(n, s->is_dup.p, d_excl_all, s->cls_obj.p, d_anchor);
    FX_LAUNCHED();
    k_dup_members<<<(unsigned)cdiv(n, 256), 256, 0, s->st>>>(n, s->is_dup.p, d_anchor, s->cluster_of.p, s->mrank.p,
                                                             s->frank.p);
    FX_LAUNCHED();
}

void launch_seal(fx_stream *s, int64_t nfeat_total, const int32_t *fmem_cls, const int32_t *fmem_cid,
                 const int64_t *foff, unsigned long long *best_bits, double *dout, int *best_pos) {
    if (nfeat_total <= 0) return;
    const PwPlan &P = *s->plan_host;
    const int per = P.n_chains + P.n_leaves + P.n_ops;
    const int threads = 256;
    size_t smem = sizeof(double) * per * (threads / 32);
    unsigned grid = (unsigned)std::min<int64_t>(cdiv(nfeat_total, threads / 32), 148 * 16);
    static const bool seal_full = getenv("FOCUS_B200_SEAL_FULL") && atoi(getenv("FOCUS_B200_SEAL_FULL"));
    if (!seal_full) {
        // screened: an fp32 pass for every member, numpy's float64 pairwise
        // order only for the candidates of each cluster's minimum
        const int D = s->cfg.dim;
        const float eps1 = (float)((double)(D + 3) * 5.960464477539063e-08 * 1.01);
        const int64_t C = s->h_ctr[C_NEXT_CID];
        DevBuf<float> c32, cn, dl;
        DevBuf<unsigned int> ub;
        c32.reserve((size_t)std::max<int64_t>(C, 1) * D);
        cn.reserve(C + 1);
        dl.reserve(nfeat_total + 1);
        ub.reserve(C + 1);
        FX_CUDA(cudaMemsetAsync(ub.p, 0xff, sizeof(unsigned int) * (C + 1), s->st));
        k_seal_c32<<<(unsigned)std::min<int64_t>(std::max<int64_t>(C, 1), 148 * 8), 256, 0, s->st>>>(C, D, s->fcent.p,
                                                                                                    c32.p, cn.p);
        const unsigned g1 = (unsigned)std::min<int64_t>(cdiv(nfeat_total, threads / 32), 148 * 16);
        const unsigned g2 = (unsigned)cdiv(nfeat_total, threads);
        if (s->cfg.feat_type == FX_F64) {
            k_seal_screen<double><<<g1, threads, 0, s->st>>>(nfeat_total, D, fmem_cls, fmem_cid, s->frow.p, c32.p, cn.p,
                                                             eps1, dl.p, ub.p);
            FX_CUDA(cudaFuncSetAttribute(k_seal_exact<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_seal_exact<double><<<g2, threads, smem, s->st>>>(nfeat_total, D, fmem_cls, fmem_cid, s->frow.p, s->fcent.p,
                                                              s->plan.p, dl.p, ub.p, best_bits, dout);
        } else {
            k_seal_screen<float><<<g1, threads, 0, s->st>>>(nfeat_total, D, fmem_cls, fmem_cid, s->frow.p, c32.p, cn.p,
                                                            eps1, dl.p, ub.p);
            FX_CUDA(cudaFuncSetAttribute(k_seal_exact<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_seal_exact<float><<<g2, threads, smem, s->st>>>(nfeat_total, D, fmem_cls, fmem_cid, s->frow.p, s->fcent.p,
                                                             s->plan.p, dl.p, ub.p, best_bits, dout);
        }
        FX_LAUNCHED();
    } else if (s->cfg.feat_type == FX_F64) {
        FX_CUDA(cudaFuncSetAttribute(k_seal_dist<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_seal_dist<double><<<grid, threads, smem, s->st>>>(nfeat_total, s->cfg.dim, fmem_cls, fmem_cid, s->frow.p,
                                                            s->fcent.p, s->plan.p, best_bits, dout);
    } else {
        FX_CUDA(cudaFuncSetAttribute(k_seal_dist<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_seal_dist<float><<<grid, threads, smem, s->st>>>(nfeat_total, s->cfg.dim, fmem_cls, fmem_cid, s->frow.p,
                                                           s->fcent.p, s->plan.p, best_bits, dout);
    }
    FX_LAUNCHED();
    k_seal_pick<<<(unsigned)cdiv(nfeat_total, 256), 256, 0, s->st>>>(nfeat_total, fmem_cid, foff, dout, best_bits,
                                                                     best_pos);
    FX_LAUNCHED();
}

}  // namespace fx
