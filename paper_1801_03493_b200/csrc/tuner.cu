// tuner.cu -- the tuner's grid evaluation on the device.
//
// _GridEvaluator._positions (tuner.py:243-256) classifies every sample object
// with every candidate profile over the FULL ranked output and takes, per
// queried class, the class's 0-based position in each object's list.  The
// list is the profile's confusion order of the emitted class with the
// emitted class spliced in at its rank (classifiers.py:136-149), so the
// position needs no list: rank from the same SeedSequence/PCG64 draw as K1a
// (first_u53 + the profile's rank thresholds, classifiers.py:59-70, 126-133),
// and the class's index in the emitted class's confusion order (host table,
// inverse permutation):
//     pos = rank - 1                      if class == emitted
//         = f        if f <  rank - 1     (f = index of class in the fillers)
//         = f + 1    otherwise;
// a class absent from the list gives 0, as argmax over an all-False row does.
// The cluster skeletons of the grid (tuner.py:211-241) run through the
// ingest engine itself (features only: no class is posted).
#include "fx_internal.cuh"

namespace fx {

__global__ void k_rank_positions(int64_t n, const int64_t *__restrict__ oid, const int32_t *__restrict__ emitted,
                                 uint64_t seed, int gt, int nthr, const uint64_t *__restrict__ thr,
                                 const int32_t *__restrict__ inv, int V1, int ncls, const int32_t *__restrict__ cls,
                                 int32_t *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int rank = 1;
    if (!gt && nthr > 0) {  // rank = 1 + #{j : thr[j] <= u}; thr is non-decreasing
        const uint64_t u = first_u53(seed, (uint64_t)oid[i], 0ull);
        int lo = 0, hi = nthr;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (thr[mid] <= u) lo = mid + 1;
            else hi = mid;
        }
        rank = 1 + lo;
    }
    const int e = emitted[i];
    for (int q = 0; q < ncls; q++) {
        const int c = cls[q];
        int pos;
        if (c == e) {
            pos = rank - 1;
        } else {
            const int f = inv[(int64_t)e * V1 + c];
            pos = f < 0 ? 0 : (f < rank - 1 ? f : f + 1);
        }
        out[(int64_t)q * n + i] = pos;
    }
}

}  // namespace fx

namespace {
template <typename T>
void h2d(T *dst, const T *src, int64_t n, cudaStream_t st) {
    if (n > 0) FX_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyHostToDevice, st));
}
template <typename T>
void d2h(T *dst, const T *src, int64_t n, cudaStream_t st) {
    if (n > 0) FX_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
}
}  // namespace

extern "C" int fx_rank_positions(int32_t device, int64_t n, const int64_t *oids, const int32_t *emitted, uint64_t seed,
                                 int32_t ground_truth, int32_t n_thr, const uint64_t *thresholds, const int32_t *inv,
                                 int32_t v1, int32_t n_classes, const int32_t *classes, int32_t *out_pos) {
    using namespace fx;
    try {
        if (n < 0 || v1 < 1 || n_classes < 0 || n_thr < 0) throw Error{FX_E_USAGE, "bad argument"};
        if (n == 0 || n_classes == 0) return FX_OK;
        if (!oids || !emitted || !inv || !classes || !out_pos || (n_thr && !thresholds))
            throw Error{FX_E_USAGE, "null argument"};
        for (int64_t i = 0; i < n; i++)
            if (emitted[i] < 0 || emitted[i] >= v1) throw Error{FX_E_USAGE, "emitted class outside the table"};
        for (int q = 0; q < n_classes; q++)
            if (classes[q] < 0 || classes[q] >= v1) throw Error{FX_E_USAGE, "queried class outside the table"};
        FX_CUDA(cudaSetDevice(device));
        init_pool(device);
        cudaStream_t st;
        FX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        {
            StreamGuard sg_(st);
            DevBuf<int64_t> o;
            DevBuf<int32_t> e, iv, c, out;
            DevBuf<uint64_t> t;
            o.reserve(n);
            e.reserve(n);
            iv.reserve((size_t)v1 * v1);
            c.reserve(n_classes);
            out.reserve((size_t)n * n_classes);
            t.reserve(n_thr + 1);
            h2d(o.p, oids, n, st);
            h2d(e.p, emitted, n, st);
            h2d(iv.p, inv, (int64_t)v1 * v1, st);
            h2d(c.p, classes, n_classes, st);
            if (n_thr) h2d(t.p, thresholds, n_thr, st);
            k_rank_positions<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(n, o.p, e.p, seed, ground_truth ? 1 : 0, n_thr, t.p,
                                                                     iv.p, v1, n_classes, c.p, out.p);
            FX_LAUNCHED();
            d2h(out_pos, out.p, (int64_t)n * n_classes, st);
            FX_CUDA(cudaStreamSynchronize(st));
        }
        FX_CUDA(cudaStreamDestroy(st));
    } catch (const Error &err) {
        set_error(err.msg);
        return err.code;
    }
    return FX_OK;
}
