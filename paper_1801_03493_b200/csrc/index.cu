// index.cu -- K3: top-K inverted index build on the device.
//
// Reference: Cluster.merge_classes (clustering.py:65-69) keeps, per cluster,
// class -> best (minimum) rank over its featured members' top-K lists;
// index.build (index.py:60-72) posts every cluster under every class of its
// class set, postings sorted ascending and unique.
//
// Device plan:
//   (a) class sets: per cluster segment of (class, rank) entries ->
//       sorted-unique classes with min rank.  Segments <= 2048 entries:
//       one CTA bitonic-sorts them in shared memory.  Larger segments:
//       chunked CTAs atomicMin into a per-segment (V+1) table (shared
//       memory, merged into global), then one CTA emits the present classes
//       in class order.
//   (b) postings: stable counting sort of the (cluster-major, class-sorted)
//       entries by class: per-chunk class histograms, one exclusive scan over
//       the class-major histogram matrix, and a warp-aggregated stable
//       scatter (__match_any_sync ranks) that preserves ascending cluster
//       order inside every class.
#include "fx_handles.cuh"

namespace fx {

constexpr int SEG_SMALL = 2048;
constexpr int CHUNK_BIG = 16384;
constexpr int POST_CH = 4096;

// entry source for ingested streams: entry e of cluster c is
// (topk[obj(fmem[foff[c] + e / K]) * K + e % K], e % K + 1)
struct EntriesFromTopk {
    const int64_t *foff;
    const int32_t *fmem_cls;
    const int64_t *cls_obj;
    const int32_t *topk;
    int K;
    __device__ int64_t seg_begin(int64_t c) const { return foff[c] * K; }
    __device__ int64_t seg_end(int64_t c) const { return foff[c + 1] * K; }
    __device__ void get(int64_t c, int64_t e, int &cls, int &rank) const {
        int64_t rel = e - foff[c] * K;
        int64_t m = foff[c] + rel / K;
        int j = (int)(rel % K);
        cls = topk[cls_obj[fmem_cls[m]] * K + j];
        rank = j + 1;
    }
};

// entry source for caller-provided class sets (fx_index_build)
struct EntriesFromCsr {
    const int64_t *off;
    const int32_t *cls;
    const int32_t *rank;
    __device__ int64_t seg_begin(int64_t c) const { return off[c]; }
    __device__ int64_t seg_end(int64_t c) const { return off[c + 1]; }
    __device__ void get(int64_t, int64_t e, int &c, int &r) const {
        c = cls[e];
        r = rank[e];
    }
};

// (a-small) sort each small segment in smem; write unique (class, min rank)
// at the segment's entry offset in tmp_cls/tmp_rank, count to cnt[c].
template <typename E>
__global__ void __launch_bounds__(512) k_classes_small(int64_t C, E src, int32_t *__restrict__ tmp_cls,
                                                       int32_t *__restrict__ tmp_rank, int32_t *__restrict__ cnt,
                                                       int32_t *__restrict__ is_big) {
    __shared__ uint32_t key[SEG_SMALL];
    __shared__ int s_n;
    for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
        const int64_t b0 = src.seg_begin(c), b1 = src.seg_end(c);
        const int64_t len = b1 - b0;
        if (len > SEG_SMALL) {
            if (threadIdx.x == 0) is_big[c] = 1;
            continue;
        }
        if (threadIdx.x == 0) is_big[c] = 0;
        int n2 = 1;
        while (n2 < len) n2 <<= 1;
        for (int i = threadIdx.x; i < n2; i += blockDim.x) {
            uint32_t k = 0xffffffffu;
            if (i < len) {
                int cl, r;
                src.get(c, b0 + i, cl, r);
                // cl < 0: a classifier emitted fewer than K classes (the
                // reference merges only the classes emitted, clustering.py:65-69)
                if (cl >= 0) k = ((uint32_t)cl << 8) | (uint32_t)(r & 0xff);
            }
            key[i] = k;
        }
        __syncthreads();
        for (int size = 2; size <= n2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                    int j = i ^ stride;
                    if (j > i) {
                        bool up = (i & size) == 0;
                        uint32_t a = key[i], b = key[j];
                        if ((a > b) == up) {
                            key[i] = b;
                            key[j] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // unique by class: first of each run has the minimum rank
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        // ordered compaction by warp 0 (ballots keep order)
        if (threadIdx.x < 32) {
            int base = 0;
            for (int i0 = 0; i0 < len; i0 += 32) {
                int i = i0 + threadIdx.x;
                bool head = i < len && key[i] != 0xffffffffu && (i == 0 || (key[i] >> 8) != (key[i - 1] >> 8));
                unsigned m = __ballot_sync(0xffffffffu, head);
                if (head) {
                    int p = base + __popc(m & ((1u << threadIdx.x) - 1u));
                    tmp_cls[b0 + p] = (int32_t)(key[i] >> 8);
                    tmp_rank[b0 + p] = (int32_t)(key[i] & 0xff);
                }
                base += __popc(m);
            }
            if (threadIdx.x == 0) cnt[c] = base;
        }
        __syncthreads();
    }
}

// (a-big, pass 1) chunked atomicMin into per-big-segment tables.
template <typename E>
__global__ void __launch_bounds__(256) k_classes_big_acc(int64_t nbig, const int32_t *__restrict__ big_list, E src,
                                                         int V1, uint32_t *__restrict__ table) {
    extern __shared__ uint32_t tab[];
    const int64_t bi = blockIdx.y;
    if (bi >= nbig) return;
    const int64_t c = big_list[bi];
    const int64_t b0 = src.seg_begin(c), b1 = src.seg_end(c);
    const int64_t lo = b0 + (int64_t)blockIdx.x * CHUNK_BIG;
    if (lo >= b1) return;
    const int64_t hi = min(b1, lo + CHUNK_BIG);
    for (int i = threadIdx.x; i < V1; i += blockDim.x) tab[i] = 0xffffffffu;
    __syncthreads();
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        int cl, r;
        src.get(c, e, cl, r);
        if (cl >= 0) atomicMin(&tab[cl], (uint32_t)r);
    }
    __syncthreads();
    uint32_t *g = table + bi * (int64_t)V1;
    for (int i = threadIdx.x; i < V1; i += blockDim.x)
        if (tab[i] != 0xffffffffu) atomicMin(&g[i], tab[i]);
}

// (a-big, pass 2) emit present classes in class order.
template <typename E>
__global__ void __launch_bounds__(1024) k_classes_big_emit(int64_t nbig, const int32_t *__restrict__ big_list, E src,
                                                           int V1, const uint32_t *__restrict__ table,
                                                           int32_t *__restrict__ tmp_cls, int32_t *__restrict__ tmp_rank,
                                                           int32_t *__restrict__ cnt) {
    const int64_t bi = blockIdx.x;
    if (bi >= nbig) return;
    const int64_t c = big_list[bi];
    const int64_t b0 = src.seg_begin(c);
    const uint32_t *g = table + bi * (int64_t)V1;
    __shared__ int wsum[32];
    __shared__ int s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int i0 = 0; i0 < V1; i0 += blockDim.x) {
        int i = i0 + threadIdx.x;
        bool present = i < V1 && g[i] != 0xffffffffu;
        unsigned m = __ballot_sync(0xffffffffu, present);
        int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (lane == 0) wsum[w] = __popc(m);
        __syncthreads();
        int before = 0;
        for (int k = 0; k < w; k++) before += wsum[k];
        if (present) {
            int p = s_base + before + __popc(m & ((1u << lane) - 1u));
            tmp_cls[b0 + p] = i;
            tmp_rank[b0 + p] = (int32_t)g[i];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); k++) t += wsum[k];
            s_base += t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) cnt[c] = s_base;
}

template <typename E>
__global__ void k_classes_copy(int64_t C, E src, const int64_t *__restrict__ out_off, const int32_t *__restrict__ tmp_cls,
                               const int32_t *__restrict__ tmp_rank, int32_t *__restrict__ cls_id,
                               int32_t *__restrict__ cls_rank) {
    for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
        const int64_t b0 = src.seg_begin(c), o0 = out_off[c], n = out_off[c + 1] - o0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            cls_id[o0 + i] = tmp_cls[b0 + i];
            cls_rank[o0 + i] = tmp_rank[b0 + i];
        }
    }
}

// entry -> owning cluster index (entries are cluster-major)
__global__ void k_entry_owner(int64_t C, const int64_t *__restrict__ off, int32_t *__restrict__ owner) {
    for (int64_t c = blockIdx.x; c < C; c += gridDim.x)
        for (int64_t e = off[c] + threadIdx.x; e < off[c + 1]; e += blockDim.x) owner[e] = (int32_t)c;
}

// (b-1) per-chunk class histograms, class-major [V1][nchunks]
__global__ void __launch_bounds__(256) k_post_hist(int64_t n, const int32_t *__restrict__ cls_id, int V1, int64_t nchunks,
                                                   int32_t *__restrict__ hist) {
    extern __shared__ int32_t h[];
    const int64_t ch = blockIdx.x;
    for (int i = threadIdx.x; i < V1; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t lo = ch * POST_CH, hi = min(n, lo + POST_CH);
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) atomicAdd(&h[cls_id[e]], 1);
    __syncthreads();
    for (int i = threadIdx.x; i < V1; i += blockDim.x) hist[(int64_t)i * nchunks + ch] = h[i];
}

// (b-2) stable warp-aggregated scatter: one warp per chunk, entries in order
__global__ void __launch_bounds__(32) k_post_scatter(int64_t n, const int32_t *__restrict__ cls_id,
                                                     const int32_t *__restrict__ cls_rank,
                                                     const int32_t *__restrict__ owner, int V1, int64_t nchunks,
                                                     const int64_t *__restrict__ hpos, int32_t *__restrict__ post_cidx,
                                                     int32_t *__restrict__ post_rank) {
    extern __shared__ int64_t base[];  // [V1] running position per class
    const int64_t ch = blockIdx.x;
    const int lane = threadIdx.x;
    for (int i = lane; i < V1; i += 32) base[i] = hpos[(int64_t)i * nchunks + ch];
    __syncwarp();
    const int64_t lo = ch * POST_CH, hi = min(n, lo + POST_CH);
    for (int64_t e0 = lo; e0 < hi; e0 += 32) {
        const int64_t e = e0 + lane;
        const bool ok = e < hi;
        const int cl = ok ? cls_id[e] : -1 - lane;
        const unsigned peers = __match_any_sync(0xffffffffu, cl);
        const int rk = __popc(peers & ((1u << lane) - 1u));
        int64_t p = 0;
        if (ok) p = base[cl] + rk;
        __syncwarp();
        if (ok) {
            post_cidx[p] = owner[e];
            post_rank[p] = cls_rank[e];
            if (rk == 0) base[cl] += __popc(peers);
        }
        __syncwarp();
    }
}

__global__ void k_post_off(int V1, int64_t nchunks, const int64_t *__restrict__ hpos, int64_t total,
                           int64_t *__restrict__ post_off) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < V1) post_off[i] = hpos[(int64_t)i * nchunks];
    if (i == V1) post_off[V1] = total;
}

// members CSR + featured CSR scatter (ingest path)
__global__ void k_member_scatter(int64_t n, const int32_t *__restrict__ cluster_of, const int32_t *__restrict__ mrank,
                                 const int32_t *__restrict__ frank, const int64_t *__restrict__ oid,
                                 const int64_t *__restrict__ fid, const int64_t *__restrict__ mem_off,
                                 const int64_t *__restrict__ foff, const int64_t *__restrict__ excl_cls,
                                 const uint8_t *__restrict__ is_dup, int64_t *__restrict__ mem_oid,
                                 int64_t *__restrict__ mem_fid, int32_t *__restrict__ fmem_cls,
                                 int32_t *__restrict__ fmem_cid) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = cluster_of[i];
    const int64_t p = mem_off[c] + mrank[i];
    mem_oid[p] = oid[i];
    mem_fid[p] = fid[i];
    if (!is_dup[i]) {
        const int64_t q = foff[c] + frank[i];
        fmem_cls[q] = (int32_t)excl_cls[i];
        fmem_cid[q] = c;
    }
}

__global__ void k_reps(int64_t C, const int64_t *__restrict__ foff, const int *__restrict__ best_pos,
                       const int32_t *__restrict__ fmem_cls, const int64_t *__restrict__ cls_obj,
                       const int64_t *__restrict__ oid, int64_t *__restrict__ reps) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C) return;
    if (foff[c + 1] == foff[c]) {
        reps[c] = -1;
        return;
    }
    reps[c] = oid[cls_obj[fmem_cls[foff[c] + best_pos[c]]]];
}

__global__ void k_iota64(int64_t n, int64_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

__global__ void k_minmax(int64_t n, const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                         unsigned long long *__restrict__ out) {
    // out[0]=min a, out[1]=max a, out[2]=min b, out[3]=max b  (biased to unsigned order)
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const unsigned long long bias = 0x8000000000000000ull;
    unsigned long long amin = ~0ull, amax = 0, bmin = ~0ull, bmax = 0;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long x = (unsigned long long)a[i] ^ bias, y = (unsigned long long)b[i] ^ bias;
        amin = x < amin ? x : amin;
        amax = x > amax ? x : amax;
        bmin = y < bmin ? y : bmin;
        bmax = y > bmax ? y : bmax;
    }
    // warp, then block reduction: one atomic per block and value (not per thread)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, amin, o);
        amin = t < amin ? t : amin;
        t = __shfl_xor_sync(0xffffffffu, amax, o);
        amax = t > amax ? t : amax;
        t = __shfl_xor_sync(0xffffffffu, bmin, o);
        bmin = t < bmin ? t : bmin;
        t = __shfl_xor_sync(0xffffffffu, bmax, o);
        bmax = t > bmax ? t : bmax;
    }
    __shared__ unsigned long long red[4][32];
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = amin;
        red[1][w] = amax;
        red[2][w] = bmin;
        red[3][w] = bmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < nw; i++) {
            amin = red[0][i] < amin ? red[0][i] : amin;
            amax = red[1][i] > amax ? red[1][i] : amax;
            bmin = red[2][i] < bmin ? red[2][i] : bmin;
            bmax = red[3][i] > bmax ? red[3][i] : bmax;
        }
        atomicMin(&out[0], amin);
        atomicMax(&out[1], amax);
        atomicMin(&out[2], bmin);
        atomicMax(&out[3], bmax);
    }
}

// duplicate cluster id check over ascending-sorted ids
__global__ void k_dup_ids(int64_t C, const int64_t *__restrict__ ids, int *__restrict__ flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > 0 && i < C && ids[i] == ids[i - 1]) atomicExch(flag, 1);
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------

int64_t scan_i32_to_i64(const int32_t *in, int64_t n, int64_t *out_excl, cudaStream_t st, int64_t *scratch_total);

template <typename E>
static void build_class_sets(fx_index *ix, E src, int64_t n_entries_in, cudaStream_t st) {
    const int64_t C = ix->C;
    const int V1 = (int)ix->V + 1;
    DevBuf<int32_t> tmp_cls, tmp_rank, cnt, is_big;
    tmp_cls.reserve(n_entries_in + 1);
    tmp_rank.reserve(n_entries_in + 1);
    cnt.reserve(C + 1);
    is_big.reserve(C + 1);
    if (C > 0) {
        unsigned g = (unsigned)std::min<int64_t>(C, 148 * 8);
        k_classes_small<E><<<g, 512, 0, st>>>(C, src, tmp_cls.p, tmp_rank.p, cnt.p, is_big.p);
        FX_LAUNCHED();
        // big segments
        std::vector<int32_t> h_big(C);
        FX_CUDA(cudaMemcpyAsync(h_big.data(), is_big.p, sizeof(int32_t) * C, cudaMemcpyDeviceToHost, st));
        FX_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> big;
        for (int64_t c = 0; c < C; c++)
            if (h_big[c]) big.push_back((int32_t)c);
        if (!big.empty()) {
            const int64_t nbig = (int64_t)big.size();
            DevBuf<int32_t> big_list;
            big_list.reserve(nbig);
            FX_CUDA(cudaMemcpyAsync(big_list.p, big.data(), sizeof(int32_t) * nbig, cudaMemcpyHostToDevice, st));
            DevBuf<uint32_t> table;
            table.reserve((size_t)nbig * V1);
            FX_CUDA(cudaMemsetAsync(table.p, 0xff, sizeof(uint32_t) * nbig * V1, st));
            int64_t max_chunks = cdiv(n_entries_in, CHUNK_BIG);
            size_t smem = sizeof(uint32_t) * V1;
            FX_CUDA(cudaFuncSetAttribute(k_classes_big_acc<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            for (int64_t off = 0; off < nbig; off += 65535) {  // grid y is limited to 65535
                const int64_t nb = std::min<int64_t>(65535, nbig - off);
                dim3 grid((unsigned)std::max<int64_t>(1, max_chunks), (unsigned)nb);
                k_classes_big_acc<E><<<grid, 256, smem, st>>>(nb, big_list.p + off, src, V1, table.p + off * V1);
                FX_LAUNCHED();
            }
            k_classes_big_emit<E><<<(unsigned)nbig, 1024, 0, st>>>(nbig, big_list.p, src, V1, table.p, tmp_cls.p,
                                                                   tmp_rank.p, cnt.p);
            FX_LAUNCHED();
            FX_CUDA(cudaStreamSynchronize(st));
        }
    }
    ix->cls_off.reserve(C + 1);
    int64_t tot_dev = 0;
    DevBuf<int64_t> tot;
    tot.reserve(1);
    int64_t total = scan_i32_to_i64(cnt.p, C, ix->cls_off.p, st, tot.p);
    (void)tot_dev;
    ix->n_cls_entries = total;
    ix->cls_id.reserve(total + 1);
    ix->cls_rank.reserve(total + 1);
    if (C > 0) {
        unsigned g = (unsigned)std::min<int64_t>(C, 148 * 8);
        k_classes_copy<E><<<g, 256, 0, st>>>(C, src, ix->cls_off.p, tmp_cls.p, tmp_rank.p, ix->cls_id.p, ix->cls_rank.p);
        FX_LAUNCHED();
    }
    FX_CUDA(cudaStreamSynchronize(st));
}

void build_postings(fx_index *ix, cudaStream_t st) {
    const int64_t n = ix->n_cls_entries;
    const int V1 = (int)ix->V + 1;
    ix->post_off.reserve(V1 + 1);
    ix->post_cidx.reserve(n + 1);
    ix->post_rank.reserve(n + 1);
    ix->n_postings = n;
    if (n == 0) {
        FX_CUDA(cudaMemsetAsync(ix->post_off.p, 0, sizeof(int64_t) * (V1 + 1), st));
    } else {
        DevBuf<int32_t> owner;
        owner.reserve(n);
        unsigned g = (unsigned)std::min<int64_t>(ix->C, 148 * 8);
        k_entry_owner<<<g, 256, 0, st>>>(ix->C, ix->cls_off.p, owner.p);
        FX_LAUNCHED();
        const int64_t nch = cdiv(n, POST_CH);
        DevBuf<int32_t> hist;
        DevBuf<int64_t> hpos, tot;
        hist.reserve((size_t)V1 * nch);
        hpos.reserve((size_t)V1 * nch + 1);
        tot.reserve(1);
        size_t smem = sizeof(int32_t) * V1;
        FX_CUDA(cudaFuncSetAttribute(k_post_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_post_hist<<<(unsigned)nch, 256, smem, st>>>(n, ix->cls_id.p, V1, nch, hist.p);
        FX_LAUNCHED();
        int64_t total = scan_i32_to_i64(hist.p, (int64_t)V1 * nch, hpos.p, st, tot.p);
        if (total != n) throw Error{FX_E_INTERNAL, "postings histogram mismatch"};
        size_t smem2 = sizeof(int64_t) * V1;
        FX_CUDA(cudaFuncSetAttribute(k_post_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        k_post_scatter<<<(unsigned)nch, 32, smem2, st>>>(n, ix->cls_id.p, ix->cls_rank.p, owner.p, V1, nch, hpos.p,
                                                         ix->post_cidx.p, ix->post_rank.p);
        FX_LAUNCHED();
        k_post_off<<<(unsigned)cdiv(V1 + 1, 256), 256, 0, st>>>(V1, nch, hpos.p, n, ix->post_off.p);
        FX_LAUNCHED();
    }
    ix->h_post_off.resize(V1 + 1);
    FX_CUDA(cudaMemcpyAsync(ix->h_post_off.data(), ix->post_off.p, sizeof(int64_t) * (V1 + 1), cudaMemcpyDeviceToHost, st));
    FX_CUDA(cudaStreamSynchronize(st));
}

void index_ranges(fx_index *ix, cudaStream_t st) {
    if (ix->n_members == 0) {
        ix->fmin = ix->omin = 0;
        ix->fmax = ix->omax = -1;
        return;
    }
    DevBuf<unsigned long long> mm;
    mm.reserve(4);
    unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
    FX_CUDA(cudaMemcpyAsync(mm.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    unsigned g = (unsigned)std::min<int64_t>(cdiv(ix->n_members, 256), 148 * 8);
    k_minmax<<<g, 256, 0, st>>>(ix->n_members, ix->mem_fid.p, ix->mem_oid.p, mm.p);
    FX_LAUNCHED();
    unsigned long long h[4];
    FX_CUDA(cudaMemcpyAsync(h, mm.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    FX_CUDA(cudaStreamSynchronize(st));
    const unsigned long long bias = 0x8000000000000000ull;
    ix->fmin = (int64_t)(h[0] ^ bias);
    ix->fmax = (int64_t)(h[1] ^ bias);
    ix->omin = (int64_t)(h[2] ^ bias);
    ix->omax = (int64_t)(h[3] ^ bias);
}

// index build from an ingested stream (finalize)
void build_index_from_stream(fx_index *ix, fx_stream *s, const int64_t *foff, const int32_t *fmem_cls,
                             int64_t nfeat_total, cudaStream_t st) {
    EntriesFromTopk src{foff, fmem_cls, s->cls_obj.p, s->topk.p, s->cfg.k};
    build_class_sets(ix, src, nfeat_total * s->cfg.k, st);
    build_postings(ix, st);
    index_ranges(ix, st);
}

// index build from caller records (fx_index_build); ids ascending
void build_index_from_csr(fx_index *ix, const int64_t *d_off, const int32_t *d_cls, const int32_t *d_rank,
                          int64_t n_entries, cudaStream_t st) {
    if (ix->C > 1) {
        DevBuf<int> flag;
        flag.reserve(1);
        FX_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
        k_dup_ids<<<(unsigned)cdiv(ix->C, 256), 256, 0, st>>>(ix->C, ix->cluster_ids.p, flag.p);
        FX_LAUNCHED();
        int h = 0;
        FX_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        FX_CUDA(cudaStreamSynchronize(st));
        if (h) throw Error{FX_E_DUPLICATE_CLUSTER_ID, "duplicate cluster id"};
    }
    EntriesFromCsr src{d_off, d_cls, d_rank};
    build_class_sets(ix, src, n_entries, st);
    build_postings(ix, st);
    index_ranges(ix, st);
}

void launch_member_scatter(fx_stream *s, int64_t n, const int64_t *mem_off, const int64_t *foff,
                           const int64_t *excl_cls, int64_t *mem_oid, int64_t *mem_fid, int32_t *fmem_cls,
                           int32_t *fmem_cid) {
    k_member_scatter<<<(unsigned)cdiv(n, 256), 256, 0, s->st>>>(n, s->cluster_of.p, s->mrank.p, s->frank.p, s->oid.p,
                                                               s->fid.p, mem_off, foff, excl_cls, s->is_dup.p, mem_oid,
                                                               mem_fid, fmem_cls, fmem_cid);
    FX_LAUNCHED();
}

void launch_reps(fx_stream *s, int64_t C, const int64_t *foff, const int *best_pos, const int32_t *fmem_cls,
                 int64_t *reps) {
    if (C <= 0) return;
    k_reps<<<(unsigned)cdiv(C, 256), 256, 0, s->st>>>(C, foff, best_pos, fmem_cls, s->cls_obj.p, s->oid.p, reps);
    FX_LAUNCHED();
}

void launch_iota64(int64_t n, int64_t *out, cudaStream_t st) {
    if (n <= 0) return;
    k_iota64<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(n, out);
    FX_LAUNCHED();
}

}  // namespace fx
