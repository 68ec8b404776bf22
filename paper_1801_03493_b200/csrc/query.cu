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

enum QCtr { Q_EXAMINED = 0, Q_MATCHED, Q_FRESH, Q_ERRPOS, Q_ERRCODE, Q_NMATCH, Q_COUNT };

// pass 1: candidate flags + first error position
__global__ void k_q_verify(int64_t seg0, int64_t nseg, const int32_t *__restrict__ post_cidx,
                           const int32_t *__restrict__ post_rank, int k_x, int batch_step,
                           const uint8_t *__restrict__ seen, const int32_t *__restrict__ rep_label, int mode,
                           int queried, int has_other, int32_t *__restrict__ cand, unsigned long long *__restrict__ qerr) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nseg) return;
    const int c = post_cidx[seg0 + i];
    int ok = post_rank[seg0 + i] <= k_x;
    if (ok && batch_step == 2 && seen[c]) ok = 0;
    cand[i] = ok;
    if (!ok) return;
    const int label = rep_label[c];
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
                          uint8_t *__restrict__ memo, uint8_t *__restrict__ seen, int batch_step, int mode, int queried,
                          int keep_label, const uint8_t *__restrict__ other_map, int V, int32_t *__restrict__ matched,
                          int64_t *__restrict__ qctr) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nseg || !cand[i]) return;
    const unsigned long long e = *qerr;
    const int64_t epos = (int64_t)(e >> 8);
    const int ecode = (int)(e & 0xff);
    const int c = post_cidx[seg0 + i];
    atomicAdd((unsigned long long *)&qctr[Q_EXAMINED], 1ull);
    if (batch_step) seen[c] = 1;
    // when the reference raised at candidate epos, only earlier candidates (and
    // the failing one when the failure comes after caching) touched the memo
    const bool touched = (e == ~0ull) || i < epos || (i == epos && ecode == 4);
    if (!touched) return;
    const int label = rep_label[c];
    const int key = rep_key[c];
    // memo: fresh iff this key was not cached before (one winner per key)
    unsigned int old = atomicOr((unsigned int *)(memo + (key & ~3)), 1u << ((key & 3) * 8));
    if (!(old & (1u << ((key & 3) * 8)))) atomicAdd((unsigned long long *)&qctr[Q_FRESH], 1ull);
    if (e != ~0ull) return;  // query raises: no result
    bool ok;
    if (mode == 1) ok = label == keep_label;
    else if (queried < 0) ok = other_map[label] != 0;
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
    if (batch_step == 1) FX_CUDA(cudaMemsetAsync(ss->seen.p, 0, ix->C ? ix->C : 1, st));
    ss->nf = ss->no = 0;
    if (nseg == 0) return;
    ss->cand.reserve(nseg);
    ss->matched.reserve(nseg);
    ss->qctr.reserve(Q_COUNT + 1);
    FX_CUDA(cudaMemsetAsync(ss->qctr.p, 0, sizeof(int64_t) * (Q_COUNT + 1), st));
    unsigned long long *qerr = (unsigned long long *)(ss->qctr.p + Q_COUNT);
    FX_CUDA(cudaMemsetAsync(qerr, 0xff, sizeof(unsigned long long), st));
    const unsigned g = (unsigned)cdiv(nseg, 256);
    k_q_verify<<<g, 256, 0, st>>>(seg0, nseg, ix->post_cidx.p, ix->post_rank.p, k_x, batch_step, ss->seen.p,
                                  ss->rep_label.p, mode, queried, ss->has_other ? 1 : 0, ss->cand.p, qerr);
    FX_LAUNCHED();
    k_q_apply<<<g, 256, 0, st>>>(seg0, nseg, ix->post_cidx.p, ss->cand.p, qerr, ss->rep_label.p, ss->rep_key.p,
                                 ss->memo.p, ss->seen.p, batch_step, mode, queried, keep_label, ss->other_map.p, V,
                                 ss->matched.p, ss->qctr.p);
    FX_LAUNCHED();
    int64_t h[Q_COUNT + 1];
    FX_CUDA(cudaMemcpyAsync(h, ss->qctr.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    FX_CUDA(cudaStreamSynchronize(st));
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
