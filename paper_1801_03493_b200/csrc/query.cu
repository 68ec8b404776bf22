// query.cu -- K4 lookup with k_x and K5 GT verification + member expansion.
//
// Reference (query.py:53-137, index.py:75-85):
//   candidates = postings[class] filtered by best rank <= k_x (ascending ids);
//   each candidate's representative is labelled by the GT classifier
//   (classifiers.py:161-165 -- a label gather), memoised per session by
//   representative object id; matched clusters contribute every member whose
//   frame lies in the inclusive time range; frames and objects are returned
//   sorted and unique.
//
// Device plan: one thread per posting entry verifies (label gather, memo,
// match); matched clusters' members set bits in frame/object bitmaps
// (atomicOr); a popcount prefix scan compacts the bitmaps into sorted unique
// id lists -- no sort needed.  Errors are reproduced at the same candidate the
// reference would raise on (first in candidate order), including the memo
// side effects of the candidates verified before it.
#include "fx_handles.cuh"

namespace fx {

enum QCtr { Q_EXAMINED = 0, Q_MATCHED, Q_FRESH, Q_ERRPOS, Q_ERRCODE, Q_NMATCH, Q_NEED, Q_COUNT };

constexpr int LBL_UNKNOWN = -5;  // label not produced yet (fx_session_create)

// pass 1: candidate flags + first error position; candidates whose label is
// not known yet are listed (the host produces them and re-issues the query)
__global__ void k_q_verify(int64_t seg0, int64_t nseg, const int32_t *__restrict__ post_cidx,
                           const int32_t *__restrict__ post_rank, int k_x, int batched,
                           const uint8_t *__restrict__ seen, const int32_t *__restrict__ rep_label, int mode,
                           int queried, int has_other, int32_t *__restrict__ cand, unsigned long long *__restrict__ qerr,
                           int64_t *__restrict__ qctr, int32_t *__restrict__ need) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nseg) return;
    const int c = post_cidx[seg0 + i];
    int ok = post_rank[seg0 + i] <= k_x;
    if (ok && batched && seen[c]) ok = 0;
    cand[i] = ok;
    if (!ok) return;
    const int label = rep_label[c];
    if (label == LBL_UNKNOWN) {
        const int p = (int)atomicAdd((unsigned long long *)&qctr[Q_NEED], 1ull);
        need[p] = c;
        return;
    }
    // error codes: 1 = MissingTrueClass (before caching), 2 = missing object (KeyError),
    // 3 = no representative, 4 = OTHER query without a specialized ingest profile (after caching)
    int code = 0;
    if (label == -2) code = 1;
    else if (label == -3) code = 2;
    else if (label == -4) code = 3;
    else if (mode == 0 && queried < 0 && !has_other) code = 4;
    if (code) atomicMin(qerr, ((unsigned long long)i << 8) | (unsigned long long)code);
}

// pass 2: apply memo / seen, count, collect matched clusters
__global__ void k_q_apply(int64_t seg0, int64_t nseg, const int32_t *__restrict__ post_cidx,
                          const int32_t *__restrict__ cand, const unsigned long long *__restrict__ qerr,
                          const int32_t *__restrict__ rep_label, const int32_t *__restrict__ rep_key,
                          uint8_t *__restrict__ memo, uint8_t *__restrict__ seen, int batched, int mode, int queried,
                          int keep_label, const uint8_t *__restrict__ other_map, int V, int32_t *__restrict__ matched,
                          int64_t *__restrict__ qctr) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nseg || !cand[i]) return;
    if (qctr[Q_NEED]) return;  // labels missing: no side effect, the host re-issues the query
    const unsigned long long e = *qerr;
    const int64_t epos = (int64_t)(e >> 8);
    const int ecode = (int)(e & 0xff);
    const int c = post_cidx[seg0 + i];
    atomicAdd((unsigned long long *)&qctr[Q_EXAMINED], 1ull);
    if (batched) seen[c] = 1;
    // when the reference raised at candidate epos, only earlier candidates (and
    // the failing one when the failure comes after caching) touched the memo
    const bool touched = (e == ~0ull) || i < epos || (i == epos && ecode == 4);
    if (!touched) return;
    const int label = rep_label[c];
    const int key = rep_key ? rep_key[c] : c;
    // memo: fresh iff this key was not cached before (one winner per key)
    unsigned int old = atomicOr((unsigned int *)(memo + (key & ~3)), 1u << ((key & 3) * 8));
    if (!(old & (1u << ((key & 3) * 8)))) atomicAdd((unsigned long long *)&qctr[Q_FRESH], 1ull);
    if (e != ~0ull) return;  // query raises: no result
    bool ok;
    if (mode == 1) ok = label == keep_label;
    else if (queried < 0) ok = (label < 0 || label >= V) ? true : other_map[label] != 0;  // map_class -> OTHER
    else ok = label == queried;
    if (ok) {
        atomicAdd((unsigned long long *)&qctr[Q_MATCHED], 1ull);
        int p = (int)atomicAdd((unsigned long long *)&qctr[Q_NMATCH], 1ull);
        matched[p] = c;
    }
}

// member expansion into bitmaps; grid (nseg, 64)
__global__ void __launch_bounds__(256) k_q_expand(const int64_t *__restrict__ qctr, const int32_t *__restrict__ matched,
                                                  const int64_t *__restrict__ mem_off, const int64_t *__restrict__ mem_oid,
                                                  const int64_t *__restrict__ mem_fid, int has_range, int64_t t0,
                                                  int64_t t1, int64_t fmin, int64_t omin, uint32_t *__restrict__ fbits,
                                                  uint32_t *__restrict__ obits) {
    const int64_t mi = blockIdx.x;
    if (mi >= qctr[Q_NMATCH]) return;
    const int c = matched[mi];
    const int64_t a = mem_off[c], b = mem_off[c + 1], len = b - a;
    const int64_t per = (len + gridDim.y - 1) / gridDim.y;
    const int64_t lo = a + per * blockIdx.y, hi = min(b, lo + per);
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
        const int64_t f = mem_fid[p];
        if (has_range && (f < t0 || f > t1)) continue;
        const int64_t fo = f - fmin, oo = mem_oid[p] - omin;
        atomicOr(&fbits[fo >> 5], 1u << (fo & 31));
        atomicOr(&obits[oo >> 5], 1u << (oo & 31));
    }
}

__global__ void k_popc(int64_t nw, const uint32_t *__restrict__ bits, int32_t *__restrict__ cnt) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nw) cnt[i] = __popc(bits[i]);
}

__global__ void k_bits_emit(int64_t nw, const uint32_t *__restrict__ bits, const int64_t *__restrict__ pos,
                            int64_t base, int64_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nw) return;
    uint32_t w = bits[i];
    int64_t p = pos[i];
    while (w) {
        int b = __ffs(w) - 1;
        out[p++] = base + i * 32 + b;
        w &= w - 1;
    }
}

int64_t scan_i32_to_i64(const int32_t *in, int64_t n, int64_t *out_excl, cudaStream_t st, int64_t *scratch_total);

static int64_t compact_bits(fx_session *ss, const uint32_t *bits, int64_t nw, int64_t base, DevBuf<int64_t> &pos,
                            DevBuf<int64_t> &out, cudaStream_t st) {
    if (nw <= 0) return 0;
    DevBuf<int32_t> cnt;
    cnt.reserve(nw);
    k_popc<<<(unsigned)cdiv(nw, 256), 256, 0, st>>>(nw, bits, cnt.p);
    FX_LAUNCHED();
    pos.reserve(nw + 1);
    DevBuf<int64_t> tot;
    tot.reserve(1);
    int64_t total = scan_i32_to_i64(cnt.p, nw, pos.p, st, tot.p);
    out.reserve(total + 1);
    if (total) {
        k_bits_emit<<<(unsigned)cdiv(nw, 256), 256, 0, st>>>(nw, bits, pos.p, base, out.p);
        FX_LAUNCHED();
    }
    (void)ss;
    return total;
}

void run_query(fx_session *ss, int class_enc, int k_x, int mode, int keep_label, int batch_step, int has_range,
               int64_t t0, int64_t t1, fx_query_result *res) {
    fx_index *ix = ss->ix;
    cudaStream_t st = ix->st;
    const int V = (int)ix->V;
    const int queried = class_enc == V ? -1 : class_enc;  // OTHER -> -1 in matching
    const int post_class = class_enc;
    const int64_t seg0 = ix->h_post_off[post_class], seg1 = ix->h_post_off[post_class + 1];
    const int64_t nseg = seg1 - seg0;
    res->n_frames = res->n_objects = res->gt_inferences = res->clusters_examined = res->clusters_matched = 0;
    res->error_cluster = -1;
    uint8_t *seen = nullptr;
    if (batch_step > 0) {
        if (batch_step > (int)ss->seen_sets.size() || !ss->seen_sets[batch_step - 1])
            throw Error{FX_E_USAGE, "batched query seen set not open"};
        seen = ss->seen_sets[batch_step - 1]->p;
    }
    ss->nf = ss->no = 0;
    ss->n_need = 0;
    if (nseg == 0) return;
    ss->cand.reserve(nseg);
    ss->matched.reserve(nseg);
    ss->need.reserve(nseg);
    ss->qctr.reserve(Q_COUNT + 1);
    FX_CUDA(cudaMemsetAsync(ss->qctr.p, 0, sizeof(int64_t) * (Q_COUNT + 1), st));
    unsigned long long *qerr = (unsigned long long *)(ss->qctr.p + Q_COUNT);
    FX_CUDA(cudaMemsetAsync(qerr, 0xff, sizeof(unsigned long long), st));
    const unsigned g = (unsigned)cdiv(nseg, 256);
    k_q_verify<<<g, 256, 0, st>>>(seg0, nseg, ix->post_cidx.p, ix->post_rank.p, k_x, seen != nullptr, seen,
                                  ss->rep_label.p, mode, queried, ss->has_other ? 1 : 0, ss->cand.p, qerr, ss->qctr.p,
                                  ss->need.p);
    FX_LAUNCHED();
    k_q_apply<<<g, 256, 0, st>>>(seg0, nseg, ix->post_cidx.p, ss->cand.p, qerr, ss->rep_label.p,
                                 ss->keyed ? ss->rep_key.p : nullptr, ss->memo.p, seen, seen != nullptr, mode, queried,
                                 keep_label, ss->other_map.p, V, ss->matched.p, ss->qctr.p);
    FX_LAUNCHED();
    int64_t h[Q_COUNT + 1];
    FX_CUDA(cudaMemcpyAsync(h, ss->qctr.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    FX_CUDA(cudaStreamSynchronize(st));
    if (h[Q_NEED]) {  // nothing was applied: the caller supplies the labels and re-issues
        ss->n_need = h[Q_NEED];
        throw Error{FX_E_NEED_LABELS, "GT labels of some representatives are needed"};
    }
    res->clusters_examined = h[Q_EXAMINED];
    res->gt_inferences = h[Q_FRESH];
    ss->gt_total += h[Q_FRESH];
    const unsigned long long e = (unsigned long long)h[Q_COUNT];
    if (e != ~0ull) {
        const int64_t epos = (int64_t)(e >> 8);
        const int code = (int)(e & 0xff);
        int32_t cidx = 0;
        FX_CUDA(cudaMemcpy(&cidx, ix->post_cidx.p + seg0 + epos, sizeof(int32_t), cudaMemcpyDeviceToHost));
        res->error_cluster = cidx;
        if (code == 1) throw Error{FX_E_MISSING_TRUE_CLASS, "representative has no true class"};
        if (code == 2) throw Error{FX_E_MISSING_OBJECT, "representative object not in objects"};
        if (code == 3) throw Error{FX_E_MISSING_OBJECT, "cluster has no representative"};
        throw Error{FX_E_UNKNOWN_CLASS, "OTHER queries need the specialized ingest profile"};
    }
    res->clusters_matched = h[Q_MATCHED];
    const int64_t nmatch = h[Q_NMATCH];
    if (nmatch == 0) return;
    const int64_t nfw = (ix->fmax - ix->fmin + 1 + 31) / 32, now = (ix->omax - ix->omin + 1 + 31) / 32;
    FX_CUDA(cudaMemsetAsync(ss->fbits.p, 0, sizeof(uint32_t) * nfw, st));
    FX_CUDA(cudaMemsetAsync(ss->obits.p, 0, sizeof(uint32_t) * now, st));
    dim3 grid((unsigned)nmatch, 64);
    k_q_expand<<<grid, 256, 0, st>>>(ss->qctr.p, ss->matched.p, ix->mem_off.p, ix->mem_oid.p, ix->mem_fid.p, has_range,
                                     t0, t1, ix->fmin, ix->omin, ss->fbits.p, ss->obits.p);
    FX_LAUNCHED();
    ss->nf = compact_bits(ss, ss->fbits.p, nfw, ix->fmin, ss->wprefix_f, ss->out_f, st);
    ss->no = compact_bits(ss, ss->obits.p, now, ix->omin, ss->wprefix_o, ss->out_o, st);
    FX_CUDA(cudaStreamSynchronize(st));
    res->n_frames = ss->nf;
    res->n_objects = ss->no;
}

__global__ void k_gather_labels(int64_t C, const int64_t *__restrict__ reps, const int32_t *__restrict__ labels,
                                int64_t base, int64_t n, int32_t *__restrict__ out) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C) return;
    const int64_t r = reps[c];
    out[c] = r < 0 ? -4 : (r - base >= 0 && r - base < n ? labels[r - base] : -3);
}

__global__ void k_scatter_labels(int64_t n, const int32_t *__restrict__ cidx, const int32_t *__restrict__ lab,
                                 int32_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[cidx[i]] = lab[i];
}

void session_gather_labels(fx_session *ss, const int32_t *labels, int64_t base, int64_t n) {
    fx_index *ix = ss->ix;
    cudaStream_t st = ix->st;
    if (ix->C == 0) return;
    DevBuf<int32_t> d;
    d.reserve(n + 1);
    if (n) FX_CUDA(cudaMemcpyAsync(d.p, labels, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    k_gather_labels<<<(unsigned)cdiv(ix->C, 256), 256, 0, st>>>(ix->C, ix->reps.p, d.p, base, n, ss->rep_label.p);
    FX_LAUNCHED();
    FX_CUDA(cudaStreamSynchronize(st));
}

void session_set_labels(fx_session *ss, int64_t n, const int32_t *cidx, const int32_t *labels) {
    fx_index *ix = ss->ix;
    cudaStream_t st = ix->st;
    if (n <= 0) return;
    for (int64_t i = 0; i < n; i++)
        if (cidx[i] < 0 || cidx[i] >= ix->C) throw Error{FX_E_USAGE, "cluster index out of range"};
    DevBuf<int32_t> d;
    d.reserve(2 * n);
    FX_CUDA(cudaMemcpyAsync(d.p, cidx, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    FX_CUDA(cudaMemcpyAsync(d.p + n, labels, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    k_scatter_labels<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(n, d.p, d.p + n, ss->rep_label.p);
    FX_LAUNCHED();
    FX_CUDA(cudaStreamSynchronize(st));
}

// index.lookup on the device: postings[class] filtered by best rank <= k_x,
// compacted in posting order (ascending cluster ids) by one CTA; ids gathered
__global__ void __launch_bounds__(1024) k_lookup(int64_t seg0, int64_t nseg, const int32_t *__restrict__ post_cidx,
                                                 const int32_t *__restrict__ post_rank, int k_x,
                                                 const int64_t *__restrict__ cluster_ids, int64_t *__restrict__ out,
                                                 int64_t *__restrict__ n_out) {
    __shared__ int wsum[32];
    __shared__ int64_t s_base;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int64_t i0 = 0; i0 < nseg; i0 += blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const bool ok = i < nseg && post_rank[seg0 + i] <= k_x;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) wsum[w] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) {
            before += k < w ? wsum[k] : 0;
            total += wsum[k];
        }
        if (ok) out[s_base + before + __popc(m & ((1u << lane) - 1u))] = cluster_ids[post_cidx[seg0 + i]];
        __syncthreads();
        if (threadIdx.x == 0) s_base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_out = s_base;
}

int64_t index_lookup(fx_index *ix, int class_enc, int k_x, int64_t *out_ids, int64_t cap) {
    cudaStream_t st = ix->st;
    const int64_t a = ix->h_post_off[class_enc], b = ix->h_post_off[class_enc + 1];
    if (b == a) return 0;
    DevBuf<int64_t> d;
    d.reserve(b - a + 1);
    k_lookup<<<1, 1024, 0, st>>>(a, b - a, ix->post_cidx.p, ix->post_rank.p, k_x, ix->cluster_ids.p, d.p, d.p + (b - a));
    FX_LAUNCHED();
    int64_t m = 0;
    FX_CUDA(cudaMemcpyAsync(&m, d.p + (b - a), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FX_CUDA(cudaStreamSynchronize(st));
    if (out_ids && m) {
        FX_CUDA(cudaMemcpyAsync(out_ids, d.p, sizeof(int64_t) * std::min(m, cap), cudaMemcpyDeviceToHost, st));
        FX_CUDA(cudaStreamSynchronize(st));
    }
    return m;
}

void session_alloc_bits(fx_session *ss) {
    fx_index *ix = ss->ix;
    const int64_t nfw = ix->n_members ? (ix->fmax - ix->fmin + 1 + 31) / 32 : 1;
    const int64_t now = ix->n_members ? (ix->omax - ix->omin + 1 + 31) / 32 : 1;
    if (nfw > (int64_t)1 << 31 || now > (int64_t)1 << 31)
        throw Error{FX_E_USAGE, "frame/object id range too sparse for the bitmap query path"};
    ss->fbits.reserve(nfw);
    ss->obits.reserve(now);
}

}  // namespace fx
