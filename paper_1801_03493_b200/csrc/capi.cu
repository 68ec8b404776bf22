// capi.cu -- the extern "C" boundary (include/focus_b200.h).
//
// Host-side orchestration only: validation (raising at the same point as the
// reference), buffer management and kernel sequencing.  All per-object and
// per-cluster work runs in the kernels of ingest.cu / index.cu / query.cu.
#include <algorithm>
#include <climits>

#include <chrono>

#include "fx_handles.cuh"

#include <mutex>

namespace fx {
const char *last_error();
int64_t launches();
void launch_dup_flags(fx_stream *s, int64_t n, const int64_t *d_fid, const double *d_sig, uint8_t *d_out);
void launch_compact(fx_stream *s, int64_t n, int64_t obj_base, int64_t cls_base, const uint8_t *d_dup,
                    const int64_t *d_excl, const char *feat_base, int compact);
void launch_fnorm(fx_stream *s, int64_t c0, int64_t nc);
void launch_rank(fx_stream *s, int64_t c0, int64_t nc, const int32_t *d_tcls, unsigned long long *d_err);
template <typename T>
void run_batches(fx_stream *s, int64_t c_begin, int64_t c_end);
void launch_final_live(fx_stream *s);
size_t resolve_smem(int Bc, const PwPlan &P);
size_t resolve_obj_bytes(int Bc, const PwPlan &P);
constexpr int FX_BMAX_DEFAULT = 8192;  // C2: 8192 is +7 %, 16384 -12 % (r02ai)
void launch_extract(int dev, int64_t n, int D, const int64_t *d_oid, const void *d_in, int in_type, int64_t ld_in,
                    double sigma, uint64_t seed, double *d_out, int64_t ld_out, unsigned long long *d_flag,
                    cudaStream_t st);
void launch_fc_head(int64_t n, int64_t c0, const char *const *frow, const int64_t *cls_obj, const float *fnorm, int D,
                    int V, int K, const float *W, const float *wnorm, const float *bias, int32_t *topk, float *conf,
                    uint8_t *flag, unsigned long long *nflag, cudaStream_t st, const float *Xdense);
void launch_row_norms(int64_t rows, int D, const float *X, float *out, cudaStream_t st);
void launch_rowptrs(int64_t rows, int64_t row_bytes, const char *base, const char **out, cudaStream_t st);
void launch_dup_members(fx_stream *s, int64_t n, const int64_t *d_excl_all, int64_t *d_anchor);
void launch_seal(fx_stream *s, int64_t nfeat_total, const int32_t *fmem_cls, const int32_t *fmem_cid,
                 const int64_t *foff, unsigned long long *best_bits, double *dout, int *best_pos);
void scan_u8_to_i64(const uint8_t *in, int64_t n, int invert, int64_t *out_excl, int64_t *d_total, cudaStream_t st);
int64_t scan_i32_to_i64(const int32_t *in, int64_t n, int64_t *out_excl, cudaStream_t st, int64_t *scratch_total);
void launch_member_scatter(fx_stream *s, int64_t n, const int64_t *mem_off, const int64_t *foff,
                           const int64_t *excl_cls, int64_t *mem_oid, int64_t *mem_fid, int32_t *fmem_cls,
                           int32_t *fmem_cid);
void launch_reps(fx_stream *s, int64_t C, const int64_t *foff, const int *best_pos, const int32_t *fmem_cls,
                 int64_t *reps);
void launch_iota64(int64_t n, int64_t *out, cudaStream_t st);
void build_index_from_stream(fx_index *ix, fx_stream *s, const int64_t *foff, const int32_t *fmem_cls,
                             int64_t nfeat_total, cudaStream_t st);
void build_index_from_csr(fx_index *ix, const int64_t *d_off, const int32_t *d_cls, const int32_t *d_rank,
                          int64_t n_entries, cudaStream_t st);
void run_query(fx_session *ss, int class_enc, int k_x, int mode, int keep_label, int batch_step, int has_range,
               int64_t t0, int64_t t1, fx_query_result *res);
void session_alloc_bits(fx_session *ss);
void launch_dup_flags_raw(int64_t n, int S, const int64_t *d_fid, const double *d_sig, double eps, uint8_t *d_out,
                          cudaStream_t st);
void session_gather_labels(fx_session *ss, const int32_t *labels, int64_t base, int64_t n);
void session_set_labels(fx_session *ss, int64_t n, const int32_t *cidx, const int32_t *labels);
int64_t index_lookup(fx_index *ix, int class_enc, int k_x, int64_t *out_ids, int64_t cap);

__global__ void k_fill_i32(int64_t n, int32_t v, int32_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = v;
}

// first classified object of the chunk: the one non-duplicate with no
// classified object before it (excl = exclusive count of classified objects)
__global__ void k_first_cls(int64_t n, const uint8_t *__restrict__ is_dup, const int64_t *__restrict__ excl,
                            unsigned long long *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !is_dup[i] && excl[i] == 0) *out = (unsigned long long)i;
}

// leading dups of a chunk attach to the previous chunk's last classified cluster
__global__ void k_lead_dups(int64_t lead, const int64_t *__restrict__ ctr, const int32_t *__restrict__ live,
                            const int32_t *__restrict__ s_cid, int32_t *__restrict__ s_size,
                            int32_t *__restrict__ cl_size) {
    __shared__ int found;
    if (threadIdx.x == 0) found = 0;
    __syncthreads();
    const int cid = (int)ctr[C_LAST_CID];
    const int L = (int)ctr[C_NLIVE];
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        int sl = live[i];
        if (s_cid[sl] == cid) {
            s_size[sl] += (int)lead;
            found = 1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && !found) cl_size[cid] += (int)lead;
}

}  // namespace fx
namespace fx {
// make the engine's main stream wait for the lagged exact chain (st2)
void chain_join(fx_stream *s) {
    for (int i = 0; i < 2; i++)
        if (s->chain_pending[i]) FX_CUDA(cudaStreamWaitEvent(s->st, s->ev_ch[i], 0));
}

__global__ void k_init_free(int64_t nslots, int32_t *__restrict__ free_stack) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nslots) free_stack[i] = (int32_t)(nslots - 1 - i);
}

}  // namespace fx

using namespace fx;

// ---------------------------------------------------------------------------
// handle destructors
// ---------------------------------------------------------------------------

void fx_stream::tstart(int phase) {
    if (!timing) return;
    int idx = -1;
    for (size_t i = 0; i < timers.size(); i++) {
        if (timers[i].phase < 0) {
            idx = (int)i;
            break;
        }
    }
    if (idx < 0) {
        Timer t;
        FX_CUDA(cudaEventCreate(&t.a));
        FX_CUDA(cudaEventCreate(&t.b));
        timers.push_back(t);
        idx = (int)timers.size() - 1;
    }
    timers[idx].phase = phase;
    FX_CUDA(cudaEventRecord(timers[idx].a, st));
    open_timer = idx;
}
void fx_stream::tstop() {
    if (!timing || open_timer < 0) return;
    FX_CUDA(cudaEventRecord(timers[open_timer].b, st));
    pending.push_back(open_timer);
    open_timer = -1;
}
void fx_stream::tcollect() {
    for (int i : pending) {
        float ms = 0.f;
        FX_CUDA(cudaEventSynchronize(timers[i].b));
        FX_CUDA(cudaEventElapsedTime(&ms, timers[i].a, timers[i].b));
        t_ms[timers[i].phase] += ms;
        timers[i].phase = -1;
    }
    pending.clear();
}

fx_stream::~fx_stream() {
    if (counted) live_engines(dev, -1);
    if (st2) cudaStreamSynchronize(st2);  // the lagged chain reads engine buffers
    for (auto &e : ev_tf)
        if (e) cudaEventDestroy(e);
    for (auto &e : ev_ch)
        if (e) cudaEventDestroy(e);
    if (h_ctr_ring) {
        for (auto &e : ring_ev)
            if (e) cudaEventSynchronize(e);
        pinned_return(h_ctr_ring);
    }
    for (auto &e : ring_ev)
        if (e) cudaEventDestroy(e);
    for (auto &t : timers) {
        if (t.a) cudaEventDestroy(t.a);
        if (t.b) cudaEventDestroy(t.b);
    }
    for (auto *b : owned_feats) delete b;
    delete plan_host;
    // the CUDA stream is destroyed by fx_stream_destroy after the members'
    // stream-ordered frees have been queued on it
}
fx_index::~fx_index() {}  // stream destroyed by fx_index_destroy (see fx_stream)
fx_session::~fx_session() {
    for (auto *b : seen_sets) delete b;
}

#define FX_GUARD(...)                                   \
    try {                                               \
        __VA_ARGS__;                                    \
        return FX_OK;                                   \
    } catch (const ::fx::Error &e_) {                   \
        ::fx::set_error(e_.msg);                        \
        return e_.code;                                 \
    } catch (const std::exception &e_) {                \
        ::fx::set_error(e_.what());                     \
        return FX_E_INTERNAL;                           \
    }

static void set_dev(int dev) { FX_CUDA(cudaSetDevice(dev)); }

template <typename T>
static void h2d(T *dst, const T *src, int64_t n, cudaStream_t st) {
    if (n > 0) FX_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyHostToDevice, st));
}
template <typename T>
static void d2h(T *dst, const T *src, int64_t n, cudaStream_t st) {
    if (n > 0 && dst) FX_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
}

extern "C" {

const char *fx_last_error(void) { return fx::last_error(); }
int fx_version(void) { return 1; }

// ---------------------------------------------------------------------------
// SM partitions (green contexts) for several engines on one device: engine i
// created after fx_device_set_partitions(dev, n) runs its streams in partition
// i mod n, so engines cannot starve each other's CTAs.  Driver
// entry points are resolved at run time (the library does not link libcuda).
// ---------------------------------------------------------------------------
namespace {
struct GreenApi {
    CUresult (*getDev)(CUdevice *, int) = nullptr;
    CUresult (*getRes)(CUdevice, CUdevResource *, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource *, unsigned int *, const CUdevResource *, CUdevResource *, unsigned int,
                      unsigned int) = nullptr;
    CUresult (*genDesc)(CUdevResourceDesc *, CUdevResource *, unsigned int) = nullptr;
    CUresult (*create)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
    CUresult (*streamCreate)(CUstream *, CUgreenCtx, unsigned int, int) = nullptr;
    bool ok = false;
};
const GreenApi &green_api() {
    static GreenApi g = [] {
        GreenApi a;
        auto get = [](const char *name, void **fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn;
        };
        a.ok = get("cuDeviceGet", (void **)&a.getDev) && get("cuDeviceGetDevResource", (void **)&a.getRes) &&
               get("cuDevSmResourceSplitByCount", (void **)&a.split) &&
               get("cuDevResourceGenerateDesc", (void **)&a.genDesc) && get("cuGreenCtxCreate", (void **)&a.create) &&
               get("cuGreenCtxStreamCreate", (void **)&a.streamCreate);
        return a;
    }();
    return g;
}
struct Partitions {
    std::mutex mu;
    std::vector<CUgreenCtx> ctx;
    std::vector<int> sms;
    int next = 0;
};
Partitions g_parts[64];
}  // namespace

extern "C" int fx_device_set_partitions(int32_t device, int32_t n_groups, int32_t *out_sms_per_group) {
    FX_GUARD({
        if (device < 0 || device >= 64 || n_groups < 0 || n_groups > 32) throw Error{FX_E_USAGE, "bad arguments"};
        Partitions &P = g_parts[device];
        std::lock_guard<std::mutex> lk(P.mu);
        P.ctx.clear();  // contexts of earlier partitions stay alive for the engines bound to them
        P.sms.clear();
        P.next = 0;
        if (out_sms_per_group) *out_sms_per_group = 0;
        if (n_groups <= 1) return FX_OK;
        const GreenApi &g = green_api();
        if (!g.ok) throw Error{FX_E_CUDA, "green contexts unavailable in this driver"};
        set_dev(device);
        FX_CUDA(cudaFree(nullptr));
        CUdevice dev;
        CUdevResource all;
        if (g.getDev(&dev, device) != CUDA_SUCCESS || g.getRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
            throw Error{FX_E_CUDA, "cuDeviceGetDevResource failed"};
        unsigned per = (all.sm.smCount / (unsigned)n_groups) & ~7u;  // multiples of 8 SMs
        if (per < 8) throw Error{FX_E_USAGE, "too many partitions for this device"};
        std::vector<CUdevResource> grp(n_groups);
        CUdevResource rem;
        unsigned ng = (unsigned)n_groups;
        if (g.split(grp.data(), &ng, &all, &rem, 0, per) != CUDA_SUCCESS || ng < (unsigned)n_groups)
            throw Error{FX_E_CUDA, "cuDevSmResourceSplitByCount failed"};
        for (unsigned i = 0; i < ng; i++) {
            CUdevResourceDesc d;
            CUgreenCtx c;
            if (g.genDesc(&d, &grp[i], 1) != CUDA_SUCCESS || g.create(&c, d, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
                throw Error{FX_E_CUDA, "cuGreenCtxCreate failed"};
            P.ctx.push_back(c);
            P.sms.push_back((int)grp[i].sm.smCount);
        }
        if (out_sms_per_group) *out_sms_per_group = P.sms.empty() ? 0 : P.sms[0];
    })
}

namespace fx {
// the partition a new engine's streams belong to (nullptr: the whole device)
static CUgreenCtx next_partition(int dev, int want) {
    Partitions &P = g_parts[dev & 63];
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.ctx.empty()) return nullptr;
    if (want > 0) return P.ctx[(size_t)(want - 1) % P.ctx.size()];
    return P.ctx[(size_t)(P.next++) % P.ctx.size()];
}
static void make_stream(cudaStream_t *st, CUgreenCtx gc, int prio) {
    if (!gc) {
        FX_CUDA(cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, prio));
        return;
    }
    CUstream cs;
    if (green_api().streamCreate(&cs, gc, CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS)
        throw Error{FX_E_CUDA, "cuGreenCtxStreamCreate failed"};
    *st = (cudaStream_t)cs;
}
}  // namespace fx
int64_t fx_kernel_launches(void) { return fx::launches(); }

int fx_stream_create(const fx_stream_config *cfg, fx_stream **out) {
    FX_GUARD({
        if (!cfg || !out) throw Error{FX_E_USAGE, "null argument"};
        if (cfg->m < 1) throw Error{FX_E_NON_POSITIVE_M, "m must be >= 1"};
        if (cfg->t < 0) throw Error{FX_E_DATA, "t must be non-negative"};
        if (cfg->k < 1 || cfg->k > 255) throw Error{FX_E_K_OUT_OF_RANGE, "k outside [1, 255]"};
        if (cfg->dim < 1 || cfg->sig_dim < 0 || cfg->vocab < 1) throw Error{FX_E_USAGE, "bad dimensions"};
        if (cfg->feat_type != FX_F32 && cfg->feat_type != FX_F64) throw Error{FX_E_USAGE, "bad feat_type"};
        set_dev(cfg->device);
        init_pool(cfg->device);
        StreamGuard sg_(nullptr);
        fx_stream *s = new fx_stream();
        try {
            s->cfg = *cfg;
            s->dev = cfg->device;
            live_engines(s->dev, +1);
            s->counted = true;
            s->esize = cfg->feat_type == FX_F64 ? 8 : 4;
            {
                const char *env = getenv("FOCUS_B200_SCREEN");
                const bool simt = env && strcmp(env, "simt") == 0;
                s->tc_screen = !simt && cfg->feat_type == FX_F32 && cfg->dim % 4 == 0;
                const char *chk = getenv("FOCUS_B200_CHECK");
                s->debug_check = chk && strcmp(chk, "1") == 0;
                const char *tm = getenv("FOCUS_B200_TIMERS");
                s->timing = tm && strcmp(tm, "1") == 0;
            }
            // the batch chain runs at the highest stream priority, the lagged
            // exact chain (st2) at the lowest: pending CTAs of the critical
            // path are scheduled ahead of the chain's
            int prio_lo = 0, prio_hi = 0;
            FX_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
            static const bool noprio = getenv("FOCUS_B200_NOPRIO") && atoi(getenv("FOCUS_B200_NOPRIO"));
            if (noprio) prio_lo = prio_hi = 0;
            CUgreenCtx gctx = next_partition(s->dev, cfg->partition);
            s->partitioned = gctx != nullptr;
            make_stream(&s->st, gctx, prio_hi);
            cur_stream() = s->st;
            const int D = cfg->dim;
            // batch capacity: up to FX_BMAX classified objects (k_resolve keeps
            // its per-object state in shared memory up to 4096, in global
            // memory above that; its windows never exceed 4096 objects)
            static const int bmax = getenv("FOCUS_B200_BMAX") ? atoi(getenv("FOCUS_B200_BMAX")) : FX_BMAX_DEFAULT;
            const int bcap = std::max(64, std::min(bmax, 16384));
            int B = cfg->batch;
            if (B <= 0) {
                int64_t b = ((int64_t)1 << 26) / std::max<int64_t>(cfg->m, 1);
                B = (int)std::min<int64_t>(bcap, std::max<int64_t>(256, b));
            }
            B = std::max(64, (std::min(B, bcap) / 64) * 64);
            s->plan_host = new PwPlan();
            build_pw_plan(D, s->plan_host);
            if (B <= 4096) {  // k_resolve keeps per-object state of the whole batch in shared memory
                while (B > 64 && resolve_smem(B, *s->plan_host) + 48 * 1024 > 227 * 1024) B -= 64;
            } else {
                s->rs_gobj.reserve(resolve_obj_bytes(B, *s->plan_host));
            }
            s->B = B;
            const int64_t max_slots_mem = (int64_t)(48e9 / (20.0 * D));  // S + S_tree + C32
            int64_t live_cap = std::min<int64_t>(cfg->m, max_slots_mem);
            s->nslots = live_cap + B + 1;
            s->ld = std::max<int64_t>(1, live_cap + 1);
            const int64_t ns = s->nslots;
            s->S.reserve((size_t)ns * D);
            s->C32.reserve((size_t)ns * D);
            for (auto *b : {&s->s_cid, &s->s_nfeat, &s->s_size, &s->s_snapq, &s->s_seedpos, &s->s_foldpos, &s->s_pend,
                            &s->s_odcol, &s->s_didx, &s->s_grp, &s->s_evicted, &s->live, &s->live_pos, &s->free_stack,
                            &s->defer_free, &s->snap_slot})
                b->reserve(ns);
            s->s_drift.reserve(ns);
            s->s_cn2.reserve(ns);
            {  // snapshot tree fold + lagged exact chain (k_tfold / k_fold on st2)
                make_stream(&s->st2, gctx, prio_lo);
                for (int i = 0; i < 2; i++) {
                    FX_CUDA(cudaEventCreateWithFlags(&s->ev_tf[i], cudaEventDisableTiming));
                    FX_CUDA(cudaEventCreateWithFlags(&s->ev_ch[i], cudaEventDisableTiming));
                }
                s->S_tree.reserve((size_t)ns * D);
                s->s_abs.reserve(ns);
                s->s_sdev.reserve(ns);
                FX_CUDA(cudaMemsetAsync(s->s_sdev.p, 0, sizeof(double) * ns, s->st));
                const size_t nd = 2 * (size_t)B + 3, gx = (size_t)cdiv(D, 128);
                s->tf_part.reserve(16 * (size_t)D + 16);
                s->tf_bcnt.reserve(gx);
                FX_CUDA(cudaMemsetAsync(s->tf_bcnt.p, 0, sizeof(int32_t) * gx, s->st));
                s->tf_cn2.reserve(nd * gx);
                s->tf_cnt.reserve(nd);
                FX_CUDA(cudaMemsetAsync(s->tf_cnt.p, 0, sizeof(int32_t) * nd, s->st));
                s->chain_epoch.reserve(1);
                s->fold_done.reserve(1);
                FX_CUDA(cudaMemsetAsync(s->chain_epoch.p, 0, sizeof(unsigned long long), s->st));
                FX_CUDA(cudaMemsetAsync(s->fold_done.p, 0, sizeof(unsigned int), s->st));
                s->tf_P.reserve((size_t)B * D);
                s->tf_PF.reserve((size_t)B);
                s->cd_meta.reserve(2 * 8 * nd);
                s->cd_off.reserve(2 * nd);
                s->cd_rows.reserve(2 * (size_t)B);
                s->cd_nd.reserve(2);
            }
            FX_CUDA(cudaMemsetAsync(s->s_cn2.p, 0, sizeof(float) * ns, s->st));
            FX_CUDA(cudaMemsetAsync(s->s_evicted.p, 0, sizeof(int32_t) * ns, s->st));
            FX_CUDA(cudaMemsetAsync(s->s_grp.p, 0xff, sizeof(int32_t) * ns, s->st));
            s->h_ctr_ring = (int64_t *)pinned_borrow(sizeof(int64_t) * 3 * C_COUNT);
            for (int i = 0; i < 3; i++) FX_CUDA(cudaEventCreateWithFlags(&s->ring_ev[i], cudaEventDisableTiming));
            s->prof.reserve(24);
            FX_CUDA(cudaMemsetAsync(s->prof.p, 0, sizeof(int64_t) * 24, s->st));
            s->ctr.reserve(C_COUNT);
            FX_CUDA(cudaMemsetAsync(s->ctr.p, 0, sizeof(int64_t) * C_COUNT, s->st));
            k_init_free<<<(unsigned)cdiv(ns, 256), 256, 0, s->st>>>(ns, s->free_stack.p);
            FX_LAUNCHED();
            int64_t nfree = ns;
            FX_CUDA(cudaMemcpyAsync(s->ctr.p + C_NFREE, &nfree, sizeof(int64_t), cudaMemcpyHostToDevice, s->st));
            s->dist.reserve((size_t)B * s->ld);
            s->dres.reserve((size_t)B * B);
            s->dod.reserve((size_t)B * B);
            for (auto *b : {&s->res_col, &s->res_pos, &s->slot_of, &s->pend_rank, &s->evict_slot, &s->evict_cid,
                            &s->pend_list, &s->pend_seg, &s->sum_slot, &s->sum_q})
                b->reserve(B + 1);
            for (auto *b : {&s->sum_d1, &s->sum_e1, &s->sum_lbr}) b->reserve(B + 1);
            for (auto *b : {&s->ev_pos, &s->ev_vic}) b->reserve(B + 1);
            {  // resolve fast path scratch (k_rfast1 / k_rfast3: 256 objects per CTA, <= 256 groups)
                const size_t nch = (size_t)cdiv(B, 256), ng = 256;
                for (auto *b : {&s->f_rank, &s->f_dup}) b->reserve(B + 1);
                s->f_P.reserve(B + 1);
                for (auto *b : {&s->f_ccnt, &s->f_cdup}) b->reserve(nch * ng);
                for (auto *b : {&s->f_csum, &s->f_cmax}) b->reserve(nch * ng);
                s->f_gi.reserve(8 * ng);
                s->f_gf.reserve(4 * ng);
                s->f_gd.reserve(8);
            }
            s->cid_slot.reserve(4 * (size_t)B);
            s->rowmin.reserve(B + 1);
            FX_CUDA(cudaMemsetAsync(s->rowmin.p, 0x7f, sizeof(int32_t) * (B + 1), s->st));
            s->snorm.reserve(s->ld);
            s->s_fjoin.reserve(ns);
            FX_CUDA(cudaMemsetAsync(s->s_fjoin.p, 0x7f, sizeof(int32_t) * ns, s->st));
            s->dirty.reserve(2 * B + 2);
            s->dirty_off.reserve(2 * B + 3);
            s->prev_sig.reserve(std::max(1, cfg->sig_dim));
            s->plan.reserve(1);
            FX_CUDA(cudaMemcpyAsync(s->plan.p, s->plan_host, sizeof(PwPlan), cudaMemcpyHostToDevice, s->st));
            FX_CUDA(cudaStreamSynchronize(s->st));
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    })
}

int fx_stream_destroy(fx_stream *s) {
    FX_GUARD({
        if (s) {
            set_dev(s->dev);
            cudaStream_t st = s->st, st2 = s->st2;
            {
                StreamGuard sg_(st);
                delete s;
            }
            if (st) cudaStreamDestroy(st);  // destroyed once its queued frees complete
            if (st2) cudaStreamDestroy(st2);
        }
    })
}

int fx_stream_set_rank_model(fx_stream *s, const fx_rank_model *rm) {
    FX_GUARD({
        if (!s || !rm) throw Error{FX_E_USAGE, "null argument"};
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        const int K = s->cfg.k, V = s->cfg.vocab;
        s->gt = rm->ground_truth;
        s->seed = rm->seed;
        s->rm_thr.reserve(K);
        s->rm_emit.reserve(V);
        s->rm_fill.reserve((size_t)(V + 1) * K);
        h2d(s->rm_thr.p, rm->thresholds, K, s->st);
        h2d(s->rm_emit.p, rm->emit_map, V, s->st);
        h2d(s->rm_fill.p, rm->fillers, (int64_t)(V + 1) * K, s->st);
        FX_CUDA(cudaStreamSynchronize(s->st));
        s->has_rm = true;
    })
}

int fx_stream_set_feature_noise(fx_stream *s, double sigma, uint64_t seed, int32_t in_type) {
    FX_GUARD({
        if (!s) throw Error{FX_E_USAGE, "null stream"};
        if (s->n_seen > 0) throw Error{FX_E_USAGE, "feature noise must be set before the first ingest"};
        if (!(sigma >= 0.0) || (in_type != FX_F32 && in_type != FX_F64))
            throw Error{FX_E_USAGE, "bad feature-noise arguments"};
        if (sigma > 0.0 && s->cfg.feat_type != FX_F64)
            throw Error{FX_E_USAGE, "feature noise needs a float64 engine (numpy's result type)"};
        if (sigma == 0.0 && in_type != s->cfg.feat_type)
            throw Error{FX_E_USAGE, "sigma = 0 copies the features: in_type must be the engine's feat_type"};
        s->has_noise = sigma > 0.0;
        s->noise_sigma = sigma;
        s->noise_seed = seed;
        s->noise_in_type = in_type;
    })
}

int fx_stream_set_fc_head(fx_stream *s, int32_t vocab, const float *W, const float *bias) {
    FX_GUARD({
        if (!s || !W) throw Error{FX_E_USAGE, "null argument"};
        if (vocab < 1 || vocab > s->cfg.vocab) throw Error{FX_E_USAGE, "fc head vocab outside [1, stream vocab]"};
        if (s->cfg.feat_type != FX_F32 || s->cfg.dim % 4 != 0)
            throw Error{FX_E_USAGE, "fc head needs float32 features with dim % 4 == 0"};
        if (s->cfg.k > 16 || s->cfg.k > vocab) throw Error{FX_E_K_OUT_OF_RANGE, "fc head: k must be <= min(16, vocab)"};
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        const int D = s->cfg.dim;
        s->fc_W.reserve((size_t)vocab * D);
        s->fc_wnorm.reserve(vocab);
        h2d(s->fc_W.p, W, (int64_t)vocab * D, s->st);
        if (bias) {
            s->fc_bias.reserve(vocab);
            h2d(s->fc_bias.p, bias, vocab, s->st);
        } else {
            s->fc_bias.release();
        }
        launch_row_norms(vocab, D, s->fc_W.p, s->fc_wnorm.p, s->st);
        FX_CUDA(cudaStreamSynchronize(s->st));
        s->fc_V = vocab;
        s->has_fc = true;
    })
}

int fx_fc_topk(int32_t device, int64_t n, int32_t dim, int32_t vocab, int32_t k, const float *feats, const float *W,
               const float *bias, int32_t *out_topk, float *out_conf, uint8_t *out_flag) {
    FX_GUARD({
        if (!feats || !W || !out_topk) throw Error{FX_E_USAGE, "null argument"};
        if (dim < 4 || dim % 4 != 0 || vocab < 1) throw Error{FX_E_USAGE, "bad shapes"};
        if (k < 1 || k > 16 || k > vocab) throw Error{FX_E_K_OUT_OF_RANGE, "k must be in [1, min(16, vocab)]"};
        if (n <= 0) return FX_OK;
        set_dev(device);
        init_pool(device);
        cudaStream_t st;
        FX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        {
            StreamGuard sg_(st);
            DevBuf<float> F, Wd, wn, bd, fn, cf;
            DevBuf<const char *> rows;
            DevBuf<int32_t> tk;
            DevBuf<uint8_t> fl;
            F.reserve((size_t)n * dim);
            Wd.reserve((size_t)vocab * dim);
            wn.reserve(vocab);
            fn.reserve(n);
            rows.reserve(n);
            tk.reserve((size_t)n * k);
            cf.reserve((size_t)n * k);
            fl.reserve(n);
            h2d(F.p, feats, n * dim, st);
            h2d(Wd.p, W, (int64_t)vocab * dim, st);
            if (bias) {
                bd.reserve(vocab);
                h2d(bd.p, bias, vocab, st);
            }
            launch_row_norms(vocab, dim, Wd.p, wn.p, st);
            launch_row_norms(n, dim, F.p, fn.p, st);
            launch_rowptrs(n, (int64_t)dim * 4, (const char *)F.p, rows.p, st);
            launch_fc_head(n, 0, rows.p, nullptr, fn.p, dim, vocab, k, Wd.p, wn.p, bias ? bd.p : nullptr, tk.p, cf.p,
                           fl.p, nullptr, st, F.p);
            d2h(out_topk, tk.p, n * k, st);
            d2h(out_conf, cf.p, n * k, st);
            d2h(out_flag, fl.p, n, st);
            FX_CUDA(cudaStreamSynchronize(st));
        }
        FX_CUDA(cudaStreamDestroy(st));
    })
}

int fx_fc_topk_device(int32_t device, void *cuda_stream, int64_t n, int32_t dim, int32_t vocab, int32_t k,
                      const float *d_feats, const float *d_W, const float *d_bias, int32_t *d_topk, float *d_conf,
                      uint8_t *d_flag) {
    FX_GUARD({
        if (!d_feats || !d_W || !d_topk) throw Error{FX_E_USAGE, "null argument"};
        if (dim < 4 || dim % 4 != 0 || vocab < 1) throw Error{FX_E_USAGE, "bad shapes"};
        if (k < 1 || k > 16 || k > vocab) throw Error{FX_E_K_OUT_OF_RANGE, "k must be in [1, min(16, vocab)]"};
        if (((uintptr_t)d_feats % 16) != 0 || ((uintptr_t)d_W % 16) != 0) throw Error{FX_E_USAGE, "unaligned rows"};
        if (n <= 0) return FX_OK;
        set_dev(device);
        init_pool(device);
        cudaStream_t st = (cudaStream_t)cuda_stream;
        StreamGuard sg_(st);
        DevBuf<float> wn, fn;
        DevBuf<const char *> rows;
        wn.reserve(vocab);
        fn.reserve(n);
        rows.reserve(n);
        launch_row_norms(vocab, dim, d_W, wn.p, st);
        launch_row_norms(n, dim, d_feats, fn.p, st);
        launch_rowptrs(n, (int64_t)dim * 4, (const char *)d_feats, rows.p, st);
        launch_fc_head(n, 0, rows.p, nullptr, fn.p, dim, vocab, k, d_W, wn.p, d_bias, d_topk, d_conf, d_flag, nullptr,
                       st, d_feats);
    })
}

// pixel_diff (ingest.py:37-47) over a sequence, no engine: a per-device
// utility stream (the drop-in `pixel_diff` of one pair, and ingest_stream's
// dup pass before the rows are marshalled)
static cudaStream_t util_stream(int device) {
    static std::mutex mu;
    static cudaStream_t st[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    const int d = device & 63;
    if (!st[d]) FX_CUDA(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    return st[d];
}

int fx_dup_flags(int32_t device, int64_t n, int32_t sig_dim, const int64_t *frame_ids, const double *sigs, double eps,
                 uint8_t *out) {
    FX_GUARD({
        if (n <= 0) return FX_OK;
        if (!frame_ids || !out || sig_dim < 0 || (sig_dim > 0 && !sigs)) throw Error{FX_E_USAGE, "bad argument"};
        set_dev(device);
        init_pool(device);
        cudaStream_t st = util_stream(device);
        StreamGuard sg_(st);
        DevBuf<int64_t> f;
        DevBuf<double> g;
        DevBuf<uint8_t> o;
        f.reserve(n);
        g.reserve((size_t)n * std::max(sig_dim, 1));
        o.reserve(n);
        h2d(f.p, frame_ids, n, st);
        if (sig_dim) h2d(g.p, sigs, n * sig_dim, st);
        launch_dup_flags_raw(n, sig_dim, f.p, g.p, eps, o.p, st);
        d2h(out, o.p, n, st);
        FX_CUDA(cudaStreamSynchronize(st));
    })
}

int fx_stream_dup_flags(fx_stream *s, int64_t n, const int64_t *frame_ids, const double *sigs, uint8_t *out) {
    FX_GUARD({
        if (!s) throw Error{FX_E_USAGE, "null stream"};
        if (n <= 0) return FX_OK;
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        const int S = s->cfg.sig_dim;
        DevBuf<int64_t> f;
        DevBuf<double> g;
        DevBuf<uint8_t> o;
        f.reserve(n);
        g.reserve((size_t)n * std::max(S, 1));
        o.reserve(n);
        h2d(f.p, frame_ids, n, s->st);
        h2d(g.p, sigs, n * S, s->st);
        launch_dup_flags(s, n, f.p, g.p, o.p);
        d2h(out, o.p, n, s->st);
        FX_CUDA(cudaStreamSynchronize(s->st));
    })
}

static void ingest_chunk(fx_stream *s, int64_t n, const int64_t *d_oid, const int64_t *d_fid, const double *d_sig,
                         const char *d_feats, const int32_t *d_tcls, const int32_t *d_topk, int compact) {
    cudaStream_t st = s->st;
    const int K = s->cfg.k, S = s->cfg.sig_dim;
    const int64_t n0 = s->n_seen, need = n0 + n;
    using hclock = std::chrono::steady_clock;
    auto hms = [](hclock::time_point a, hclock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto h0 = hclock::now();
    // per-object arrays
    s->oid.grow(need, n0, st);
    s->fid.grow(need, n0, st);
    s->is_dup.grow(need, n0, st);
    s->topk.grow((size_t)need * K, (size_t)n0 * K, st);
    s->cluster_of.grow(need, n0, st);
    s->mrank.grow(need, n0, st);
    s->frank.grow(need, n0, st);
    const auto h1 = hclock::now();
    s->t_ms[12] += hms(h0, h1);
    FX_CUDA(cudaMemcpyAsync(s->oid.p + n0, d_oid, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
    FX_CUDA(cudaMemcpyAsync(s->fid.p + n0, d_fid, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
    // K0
    s->tstart(0);
    launch_dup_flags(s, n, d_fid, d_sig, s->is_dup.p + n0);
    s->has_prev = true;
    FX_CUDA(cudaMemcpyAsync(&s->prev_fid, d_fid + (n - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (S > 0)
        FX_CUDA(cudaMemcpyAsync(s->prev_sig.p, d_sig + (n - 1) * S, sizeof(double) * S, cudaMemcpyDeviceToDevice, st));
    // classified compaction
    DevBuf<int64_t> excl, tot;
    excl.reserve(n + 1);
    tot.reserve(1);
    scan_u8_to_i64(s->is_dup.p + n0, n, 1, excl.p, tot.p, st);
    int64_t nc = 0;
    FX_CUDA(cudaMemcpyAsync(&nc, tot.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DevBuf<unsigned long long> first;
    first.reserve(1);
    FX_CUDA(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), st));
    k_first_cls<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(n, s->is_dup.p + n0, excl.p, first.p);
    FX_LAUNCHED();
    unsigned long long h_first = 0;
    FX_CUDA(cudaMemcpyAsync(&h_first, first.p, sizeof(h_first), cudaMemcpyDeviceToHost, st));
    s->tstop();
    FX_CUDA(cudaStreamSynchronize(st));
    const auto h2 = hclock::now();
    s->t_ms[13] += hms(h1, h2);
    s->tstart(0);
    const int64_t lead = h_first == ~0ull ? n : (int64_t)h_first;
    const int64_t c0 = s->n_cls, cneed = c0 + nc;
    s->cls_obj.grow(cneed, c0, st);
    s->frow.grow(cneed, c0, st);
    s->fnorm.grow(cneed, c0, st);
    s->dup_run.grow(cneed, c0, st);
    if (lead > 0 && c0 > 0) {
        // dups at the head of the chunk follow the previous chunk's last classified object
        chain_join(s);  // an evicted cluster's size is written by the chain
        k_lead_dups<<<1, 256, 0, st>>>(lead, s->ctr.p, s->live.p, s->s_cid.p, s->s_size.p, s->cl_size.p);
        FX_LAUNCHED();
    }
    if (((uintptr_t)d_feats % 16) != 0 || ((int64_t)s->cfg.dim * s->esize) % 16 != 0) s->rows_aligned16 = false;
    launch_compact(s, n, n0, c0, s->is_dup.p + n0, excl.p, d_feats, compact);
    s->arows = compact ? nc : n;
    if (!s->tc_screen || s->has_fc) launch_fnorm(s, c0, nc);  // else the TC screen computes the batch's norms
    // K1: top-K
    if (!d_topk && s->has_fc) {
        if (!s->rows_aligned16) throw Error{FX_E_USAGE, "fc head needs 16-byte aligned feature rows"};
        launch_fc_head(nc, c0, s->frow.p, s->cls_obj.p, s->fnorm.p, s->cfg.dim, s->fc_V, K, s->fc_W.p, s->fc_wnorm.p,
                       s->fc_bias.n ? s->fc_bias.p : nullptr, s->topk.p, nullptr, nullptr,
                       (unsigned long long *)(s->ctr.p + C_FCFLAG), st,
                       s->a_compact && s->esize == 4 ? (const float *)s->abase + (c0 - s->a_cbase) * s->cfg.dim
                                                       : nullptr);
        s->tstop();
    } else if (d_topk) {
        FX_CUDA(cudaMemcpyAsync(s->topk.p + n0 * K, d_topk, sizeof(int32_t) * n * K, cudaMemcpyDeviceToDevice, st));
        s->tstop();
    } else {
        if (!s->has_rm) throw Error{FX_E_USAGE, "no rank model set and no top-K given"};
        DevBuf<unsigned long long> err;
        err.reserve(1);
        FX_CUDA(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), st));
        // true_class indexed by global object index: shift the base pointer
        launch_rank(s, c0, nc, d_tcls - n0, err.p);
        s->tstop();
        unsigned long long h = 0;
        FX_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        FX_CUDA(cudaStreamSynchronize(st));
        if (h != ~0ull) {
            int64_t bad = 0;
            FX_CUDA(cudaMemcpy(&bad, s->oid.p + h, sizeof(int64_t), cudaMemcpyDeviceToHost));
            throw Error{FX_E_MISSING_TRUE_CLASS, "object " + std::to_string(bad) + " has no true class"};
        }
    }
    s->t_ms[14] += hms(h2, hclock::now());
    // K2
    if (s->cfg.feat_type == FX_F64)
        run_batches<double>(s, c0, cneed);
    else
        run_batches<float>(s, c0, cneed);
    s->n_seen = need;
    s->n_cls = cneed;
}

static int ingest_common(fx_stream *s, int64_t n, const int64_t *object_ids, const int64_t *frame_ids,
                         const double *sigs, const void *feats, const int32_t *true_class, const int32_t *topk,
                         int32_t flags, bool device, int64_t n_rows = -1) {
    FX_GUARD({
        if (!s) throw Error{FX_E_USAGE, "null stream"};
        if (s->finalized) throw Error{FX_E_USAGE, "stream already finalized"};
        if (n < 0) throw Error{FX_E_USAGE, "negative n"};
        if (n == 0) return FX_OK;
        if (!true_class && !topk && !s->has_fc) throw Error{FX_E_USAGE, "need true_class, topk or an fc head"};
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        cudaStream_t st = s->st;
        const int D = s->cfg.dim, S = s->cfg.sig_dim, K = s->cfg.k;
        const bool compact = flags & FX_FEATS_COMPACT;
        if (s->has_noise && (device || !compact))
            throw Error{FX_E_USAGE, "feature noise: host fx_ingest with FX_FEATS_COMPACT rows only"};
        if (device) {
            ingest_chunk(s, n, object_ids, frame_ids, sigs, (const char *)feats, true_class, topk, compact);
        } else {
            // host buffers: the copies run on a side stream in chunks of CH
            // objects and the engine consumes chunk k as soon as it has landed,
            // so PCIe transfer of later chunks overlaps the ingest of earlier
            // ones (pinned host memory makes the copies truly asynchronous).
            // Compact features (FX_FEATS_COMPACT: rows of the classified
            // objects only, as a cheap CNN emits them after pixel
            // differencing) need the duplicate flags first to place the
            // chunk boundaries in the row array: the small per-object arrays
            // go up first and K0 runs on them.
            // chunk of CH objects (~FOCUS_B200_H2D_MB MB of feature rows, default 256):
            // the GPU is far ahead of PCIe, so what is left after the last
            // copy lands (that chunk's ingest + finalize) is the e2e tail
            static const int64_t ch_mb = getenv("FOCUS_B200_H2D_MB") ? std::max(16, atoi(getenv("FOCUS_B200_H2D_MB"))) : 256;
            const int64_t CH = std::max<int64_t>(4096, (ch_mb << 20) / std::max<int64_t>(1, (int64_t)D * s->esize));
            const int nch = (int)cdiv(n, CH);
            DevBuf<int64_t> o, f;
            DevBuf<double> g;
            DevBuf<int32_t> tc, tk;
            DevBuf<int64_t> noise_oid;  // feature noise: classified objects' ids
            DevBuf<char> raw;           // feature noise: one chunk of raw rows
            o.reserve(n);
            f.reserve(n);
            g.reserve((size_t)n * std::max(S, 1));
            if (true_class) tc.reserve(n);
            if (topk) tk.reserve((size_t)n * K);
            std::vector<int64_t> row0(nch + 1, 0);  // first feature row of each chunk
            // the row count is known (fx_ingest_rows): the feature rows start
            // crossing PCIe at once, in row chunks, while the per-object arrays
            // go up and K0 places the object chunks' boundaries
            const bool early = compact && n_rows >= 0 && !s->has_noise;
            const size_t rbe = (size_t)D * s->esize;
            DevBuf<char> *fbe = nullptr;
            cudaStream_t cste = nullptr;
            std::vector<cudaEvent_t> evr;
            const int64_t nrch = early ? cdiv(std::max<int64_t>(n_rows, 1), CH) : 0;
            struct EarlyGuard {
                cudaStream_t *cs;
                std::vector<cudaEvent_t> *ev;
                ~EarlyGuard() {
                    if (*cs) cudaStreamSynchronize(*cs);
                    for (auto e : *ev)
                        if (e) cudaEventDestroy(e);
                    if (*cs) cudaStreamDestroy(*cs);
                }
            } early_guard_{&cste, &evr};
            if (early) {
                fbe = new DevBuf<char>();
                s->owned_feats.push_back(fbe);
                fbe->reserve((size_t)std::max<int64_t>(1, n_rows) * rbe);
                if (true_class) h2d(tc.p, true_class, n, st);
                if (topk) h2d(tk.p, topk, n * K, st);
            }
            if (compact) {
                h2d(o.p, object_ids, n, st);
                h2d(f.p, frame_ids, n, st);
                h2d(g.p, sigs, n * S, st);
                if (early) {  // the feature rows queue behind the small per-object copies
                    FX_CUDA(cudaStreamCreateWithFlags(&cste, cudaStreamNonBlocking));
                    evr.assign((size_t)nrch + 1, nullptr);
                    FX_CUDA(cudaEventCreateWithFlags(&evr[nrch], cudaEventDisableTiming));
                    FX_CUDA(cudaEventRecord(evr[nrch], st));  // allocation and small copies first
                    FX_CUDA(cudaStreamWaitEvent(cste, evr[nrch], 0));
                    for (int64_t j = 0; j < nrch; j++) {
                        const int64_t r0 = j * CH, nr = std::min<int64_t>(CH, n_rows - r0);
                        if (nr > 0)
                            FX_CUDA(cudaMemcpyAsync(fbe->p + (size_t)r0 * rbe, (const char *)feats + (size_t)r0 * rbe,
                                                    (size_t)nr * rbe, cudaMemcpyHostToDevice, cste));
                        FX_CUDA(cudaEventCreateWithFlags(&evr[j], cudaEventDisableTiming));
                        FX_CUDA(cudaEventRecord(evr[j], cste));
                    }
                }
                DevBuf<uint8_t> dup;
                dup.reserve(n);
                launch_dup_flags(s, n, f.p, g.p, dup.p);
                std::vector<uint8_t> hd(n);
                d2h(hd.data(), dup.p, n, st);
                FX_CUDA(cudaStreamSynchronize(st));
                for (int c = 0; c < nch; c++) {
                    int64_t r = 0;
                    for (int64_t i = c * CH, e = std::min<int64_t>(n, (c + 1) * CH); i < e; i++) r += hd[i] ? 0 : 1;
                    row0[c + 1] = row0[c] + r;
                }
                if (s->has_noise) {  // object ids of the classified rows (extract_feature's rng key)
                    std::vector<int64_t> co;
                    co.reserve((size_t)row0[nch]);
                    for (int64_t i = 0; i < n; i++)
                        if (!hd[i]) co.push_back(object_ids[i]);
                    noise_oid.reserve(std::max<size_t>(1, co.size()));
                    h2d(noise_oid.p, co.data(), (int64_t)co.size(), st);
                    FX_CUDA(cudaStreamSynchronize(st));  // co is pageable and goes out of scope
                }
            } else {
                for (int c = 0; c < nch; c++) row0[c + 1] = std::min<int64_t>(n, (int64_t)(c + 1) * CH);
            }
            if (early) {
                if (row0[nch] != n_rows)
                    throw Error{FX_E_USAGE, "feature rows (" + std::to_string(n_rows) + ") != classified objects (" +
                                                std::to_string(row0[nch]) + ")"};
                for (int c = 0; c < nch; c++) {
                    const int64_t a = c * CH, m = std::min<int64_t>(CH, n - a);
                    if (row0[c + 1] > row0[c])
                        FX_CUDA(cudaStreamWaitEvent(st, evr[(size_t)((row0[c + 1] - 1) / CH)], 0));
                    ingest_chunk(s, m, o.p + a, f.p + a, g.p + a * S, fbe->p + (size_t)row0[c] * rbe,
                                 true_class ? tc.p + a : nullptr, topk ? tk.p + a * K : nullptr, 1);
                }
                FX_CUDA(cudaStreamSynchronize(st));
                return FX_OK;
            }
            // feature rows stay resident until finalize (the reference retains
            // member features until seal, clustering.py:71-83)
            auto *fb = new DevBuf<char>();
            s->owned_feats.push_back(fb);
            fb->reserve((size_t)std::max<int64_t>(1, row0[nch]) * D * s->esize);
            cudaStream_t cst = nullptr;
            FX_CUDA(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
            std::vector<cudaEvent_t> ev(nch + 1, nullptr);
            try {
                FX_CUDA(cudaEventCreateWithFlags(&ev[nch], cudaEventDisableTiming));
                FX_CUDA(cudaEventRecord(ev[nch], st));  // the allocations above are ordered before the copies
                FX_CUDA(cudaStreamWaitEvent(cst, ev[nch], 0));
                const size_t rb = (size_t)D * s->esize;
                for (int c = 0; c < nch; c++) {
                    const int64_t a = c * CH, m = std::min<int64_t>(CH, n - a);
                    if (!compact) {
                        h2d(o.p + a, object_ids + a, m, cst);
                        h2d(f.p + a, frame_ids + a, m, cst);
                        h2d(g.p + a * S, sigs + a * S, m * S, cst);
                    }
                    if (true_class) h2d(tc.p + a, true_class + a, m, cst);
                    if (topk) h2d(tk.p + a * K, topk + a * K, m * K, cst);
                    const int64_t r0 = row0[c], nr = row0[c + 1] - row0[c];
                    if (nr > 0 && s->has_noise) {
                        // raw rows -> staging, extract_feature (classifiers.py:152-158) -> engine rows
                        const size_t ib = (size_t)D * (s->noise_in_type == FX_F32 ? 4 : 8);
                        if (raw.n < (size_t)nr * ib) {
                            StreamGuard sg2_(cst);
                            raw.reserve((size_t)CH * ib);
                        }
                        FX_CUDA(cudaMemcpyAsync(raw.p, (const char *)feats + (size_t)r0 * ib, (size_t)nr * ib,
                                                cudaMemcpyHostToDevice, cst));
                        launch_extract(s->dev, nr, D, noise_oid.p + r0, raw.p, s->noise_in_type, D, s->noise_sigma,
                                       s->noise_seed, (double *)(fb->p + (size_t)r0 * rb), D,
                                       (unsigned long long *)(s->ctr.p + C_NOISEFLAG), cst);
                    } else if (nr > 0) {
                        FX_CUDA(cudaMemcpyAsync(fb->p + (size_t)r0 * rb, (const char *)feats + (size_t)r0 * rb,
                                                (size_t)nr * rb, cudaMemcpyHostToDevice, cst));
                    }
                    FX_CUDA(cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming));
                    FX_CUDA(cudaEventRecord(ev[c], cst));
                }
                for (int c = 0; c < nch; c++) {
                    const int64_t a = c * CH, m = std::min<int64_t>(CH, n - a);
                    FX_CUDA(cudaStreamWaitEvent(st, ev[c], 0));
                    ingest_chunk(s, m, o.p + a, f.p + a, g.p + a * S, fb->p + (size_t)row0[c] * rb,
                                 true_class ? tc.p + a : nullptr, topk ? tk.p + a * K : nullptr, compact ? 1 : 0);
                }
                FX_CUDA(cudaStreamSynchronize(st));
            } catch (...) {
                cudaStreamSynchronize(cst);
                for (auto e : ev)
                    if (e) cudaEventDestroy(e);
                cudaStreamDestroy(cst);
                throw;
            }
            for (auto e : ev) cudaEventDestroy(e);
            FX_CUDA(cudaStreamDestroy(cst));
        }
    })
}

int fx_ingest(fx_stream *s, int64_t n, const int64_t *object_ids, const int64_t *frame_ids, const double *sigs,
              const void *feats, const int32_t *true_class, const int32_t *topk, int32_t flags) {
    return ingest_common(s, n, object_ids, frame_ids, sigs, feats, true_class, topk, flags, false);
}

int fx_ingest_rows(fx_stream *s, int64_t n, const int64_t *object_ids, const int64_t *frame_ids, const double *sigs,
                   const void *feats, int64_t n_feat_rows, const int32_t *true_class, const int32_t *topk) {
    if (n_feat_rows < 0) {
        set_error("fx_ingest_rows: negative row count");
        return FX_E_USAGE;
    }
    return ingest_common(s, n, object_ids, frame_ids, sigs, feats, true_class, topk, FX_FEATS_COMPACT, false,
                         n_feat_rows);
}

int fx_ingest_device(fx_stream *s, int64_t n, const int64_t *object_ids, const int64_t *frame_ids, const double *sigs,
                     const void *feats, const int32_t *true_class, const int32_t *topk, int32_t flags) {
    return ingest_common(s, n, object_ids, frame_ids, sigs, feats, true_class, topk, flags, true);
}

int fx_finalize(fx_stream *s, fx_index **out, fx_ingest_report *rep) {
    FX_GUARD({
        if (!s || !out) throw Error{FX_E_USAGE, "null argument"};
        if (s->finalized) throw Error{FX_E_USAGE, "stream already finalized"};
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        cudaStream_t st = s->st;
        const int D = s->cfg.dim;
        chain_join(s);  // final centroids read the exact sums
        FX_CUDA(cudaMemcpyAsync(s->h_ctr, s->ctr.p, sizeof(int64_t) * C_COUNT, cudaMemcpyDeviceToHost, st));
        FX_CUDA(cudaStreamSynchronize(st));
        if (s->h_ctr[C_ERR]) throw Error{FX_E_INTERNAL, "resolve: candidate list overflow"};
        const int64_t C = s->h_ctr[C_NEXT_CID], n = s->n_seen, nc = s->n_cls;
        if (C > s->cl_cap) {
            s->fcent.grow((size_t)C * D, (size_t)s->cl_cap * D, st);
            s->cl_nfeat.grow(C, s->cl_cap, st);
            s->cl_size.grow(C, s->cl_cap, st);
            s->cl_cap = C;
        }
        launch_final_live(s);
        fx_index *ix = new fx_index();
        try {
            ix->dev = s->dev;
            ix->st = st;
            ix->C = C;
            ix->D = D;
            ix->V = s->cfg.vocab;
            ix->K = s->cfg.k;
            ix->n_members = n;
            ix->has_centroids = true;
            DevBuf<int64_t> excl_all, tot, anchor, foff;
            excl_all.reserve(n + 1);
            tot.reserve(1);
            anchor.reserve(n + 1);
            if (n > 0) {
                scan_u8_to_i64(s->is_dup.p, n, 1, excl_all.p, tot.p, st);
                launch_dup_members(s, n, excl_all.p, anchor.p);
            }
            ix->mem_off.reserve(C + 1);
            foff.reserve(C + 1);
            int64_t nm = scan_i32_to_i64(s->cl_size.p, C, ix->mem_off.p, st, tot.p);
            int64_t nf = scan_i32_to_i64(s->cl_nfeat.p, C, foff.p, st, tot.p);
            if (nm != n || nf != nc) throw Error{FX_E_INTERNAL, "member accounting mismatch"};
            ix->mem_oid.reserve(n + 1);
            ix->mem_fid.reserve(n + 1);
            DevBuf<int32_t> fmem_cls, fmem_cid;
            fmem_cls.reserve(nc + 1);
            fmem_cid.reserve(nc + 1);
            if (n > 0)
                launch_member_scatter(s, n, ix->mem_off.p, foff.p, excl_all.p, ix->mem_oid.p, ix->mem_fid.p,
                                      fmem_cls.p, fmem_cid.p);
            // deferred seal
            DevBuf<unsigned long long> best_bits;
            DevBuf<double> dout;
            DevBuf<int> best_pos;
            best_bits.reserve(C + 1);
            best_pos.reserve(C + 1);
            dout.reserve(nc + 1);
            FX_CUDA(cudaMemsetAsync(best_bits.p, 0xff, sizeof(unsigned long long) * (C + 1), st));
            FX_CUDA(cudaMemsetAsync(best_pos.p, 0x7f, sizeof(int) * (C + 1), st));
            s->tstart(4);
            launch_seal(s, nc, fmem_cls.p, fmem_cid.p, foff.p, best_bits.p, dout.p, best_pos.p);
            s->tstop();
            ix->reps.reserve(C + 1);
            launch_reps(s, C, foff.p, best_pos.p, fmem_cls.p, ix->reps.p);
            ix->cluster_ids.reserve(C + 1);
            launch_iota64(C, ix->cluster_ids.p, st);
            std::swap(ix->centroids.p, s->fcent.p);
            std::swap(ix->centroids.n, s->fcent.n);
            s->cl_cap = 0;
            s->tstart(5);
            build_index_from_stream(ix, s, foff.p, fmem_cls.p, nc, st);
            s->tstop();
            FX_CUDA(cudaStreamSynchronize(st));
            s->tcollect();
        } catch (...) {
            ix->st = nullptr;
            delete ix;
            throw;
        }
        s->finalized = true;
        if (rep) {
            rep->objects_seen = n;
            rep->objects_classified = nc;
            rep->clusters_emitted = C;
            rep->distance_computations = s->h_ctr[C_DC];
            rep->gt_invocations = 0;
            rep->exact_rechecks = s->h_ctr[C_EXACT];
        }
        // the index shares the stream's CUDA stream; give it its own
        FX_CUDA(cudaStreamCreateWithFlags(&ix->st, cudaStreamNonBlocking));
        ix->owns_stream = true;
        *out = ix;
    })
}

int fx_stream_object_results(fx_stream *s, int32_t *cluster_of, uint8_t *is_dup, int32_t *topk) {
    FX_GUARD({
        if (!s) throw Error{FX_E_USAGE, "null stream"};
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        const int64_t n = s->n_seen;
        d2h(cluster_of, s->cluster_of.p, n, s->st);
        d2h(is_dup, s->is_dup.p, n, s->st);
        d2h(topk, s->topk.p, n * s->cfg.k, s->st);
        FX_CUDA(cudaStreamSynchronize(s->st));
    })
}

int fx_stream_timings(fx_stream *s, double *out, int n) {
    FX_GUARD({
        if (!s || !out) throw Error{FX_E_USAGE, "null argument"};
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        s->tcollect();
        for (int i = 0; i < n && i < 16; i++) out[i] = s->t_ms[i];
    })
}

int fx_stream_set_timing(fx_stream *s, int32_t on) {
    FX_GUARD({
        if (!s) throw Error{FX_E_USAGE, "null stream"};
        s->timing = on != 0;
    })
}

int fx_stream_counters(fx_stream *s, int64_t *out, int n) {
    FX_GUARD({
        if (!s || !out) throw Error{FX_E_USAGE, "null argument"};
        set_dev(s->dev);
        StreamGuard sg_(s->st);
        FX_CUDA(cudaMemcpyAsync(s->h_ctr, s->ctr.p, sizeof(int64_t) * C_COUNT, cudaMemcpyDeviceToHost, s->st));
        FX_CUDA(cudaStreamSynchronize(s->st));
        FX_CUDA(cudaStreamSynchronize(s->st2));  // fold profile counters
        for (int i = 0; i < n && i < C_COUNT; i++) out[i] = s->h_ctr[i];
        if (n > C_COUNT) {
            int64_t pr[24];
            FX_CUDA(cudaMemcpy(pr, s->prof.p, sizeof(pr), cudaMemcpyDeviceToHost));
            for (int i = C_COUNT; i < n && i < C_COUNT + 24; i++) out[i] = pr[i - C_COUNT];
        }
    })
}

void *fx_stream_cuda_stream(fx_stream *s) { return s ? (void *)s->st : nullptr; }

int fx_index_sizes_get(fx_index *ix, fx_index_sizes *o) {
    FX_GUARD({
        if (!ix || !o) throw Error{FX_E_USAGE, "null argument"};
        o->n_clusters = ix->C;
        o->dim = ix->D;
        o->n_members = ix->n_members;
        o->n_class_entries = ix->n_cls_entries;
        o->n_postings = ix->n_postings;
        o->vocab = ix->V;
        o->k = ix->K;
        o->has_centroids = ix->has_centroids ? 1 : 0;
    })
}

int fx_index_export(fx_index *ix, int64_t *cluster_ids, double *centroids, int64_t *reps, int64_t *mem_off,
                    int64_t *mem_oid, int64_t *mem_fid, int64_t *cls_off, int32_t *cls_id, int32_t *cls_rank,
                    int64_t *post_off, int64_t *post_cluster) {
    FX_GUARD({
        if (!ix) throw Error{FX_E_USAGE, "null index"};
        set_dev(ix->dev);
        StreamGuard sg_(ix->st);
        cudaStream_t st = ix->st;
        const int64_t C = ix->C;
        d2h(cluster_ids, ix->cluster_ids.p, C, st);
        if (centroids && ix->has_centroids) d2h(centroids, ix->centroids.p, C * ix->D, st);
        d2h(reps, ix->reps.p, C, st);
        d2h(mem_off, ix->mem_off.p, C + 1, st);
        d2h(mem_oid, ix->mem_oid.p, ix->n_members, st);
        d2h(mem_fid, ix->mem_fid.p, ix->n_members, st);
        d2h(cls_off, ix->cls_off.p, C + 1, st);
        d2h(cls_id, ix->cls_id.p, ix->n_cls_entries, st);
        d2h(cls_rank, ix->cls_rank.p, ix->n_cls_entries, st);
        d2h(post_off, ix->post_off.p, ix->V + 2, st);
        if (post_cluster && ix->n_postings) {
            std::vector<int32_t> tmp(ix->n_postings);
            std::vector<int64_t> ids(C);
            d2h(tmp.data(), ix->post_cidx.p, ix->n_postings, st);
            d2h(ids.data(), ix->cluster_ids.p, C, st);
            FX_CUDA(cudaStreamSynchronize(st));
            for (int64_t i = 0; i < ix->n_postings; i++) post_cluster[i] = ids[tmp[i]];
        }
        FX_CUDA(cudaStreamSynchronize(st));
    })
}

int fx_index_build(int64_t C, int32_t vocab, int32_t k, int32_t dim, int32_t device, const int64_t *cluster_ids,
                   const double *centroids, const int64_t *reps, const int64_t *mem_off, const int64_t *mem_oid,
                   const int64_t *mem_fid, const int64_t *cls_off, const int32_t *cls_id, const int32_t *cls_rank,
                   fx_index **out) {
    FX_GUARD({
        if (!out || C < 0) throw Error{FX_E_USAGE, "bad argument"};
        if (k < 1 || k > 255) throw Error{FX_E_K_OUT_OF_RANGE, "k outside [1, 255]"};
        for (int64_t i = 1; i < C; i++)
            if (cluster_ids[i] < cluster_ids[i - 1]) throw Error{FX_E_USAGE, "cluster ids must be ascending"};
        set_dev(device);
        init_pool(device);
        StreamGuard sg_(nullptr);
        fx_index *ix = new fx_index();
        try {
            ix->dev = device;
            FX_CUDA(cudaStreamCreateWithFlags(&ix->st, cudaStreamNonBlocking));
            ix->owns_stream = true;
            cudaStream_t st = ix->st;
            cur_stream() = st;
            ix->C = C;
            ix->D = dim;
            ix->V = vocab;
            ix->K = k;
            const int64_t nm = C ? mem_off[C] : 0, ne = C ? cls_off[C] : 0;
            ix->n_members = nm;
            ix->cluster_ids.reserve(C + 1);
            h2d(ix->cluster_ids.p, cluster_ids, C, st);
            ix->has_centroids = centroids != nullptr;
            if (centroids) {
                ix->centroids.reserve((size_t)C * dim + 1);
                h2d(ix->centroids.p, centroids, C * dim, st);
            }
            ix->reps.reserve(C + 1);
            h2d(ix->reps.p, reps, C, st);
            ix->mem_off.reserve(C + 1);
            h2d(ix->mem_off.p, mem_off, C + 1, st);
            ix->mem_oid.reserve(nm + 1);
            ix->mem_fid.reserve(nm + 1);
            h2d(ix->mem_oid.p, mem_oid, nm, st);
            h2d(ix->mem_fid.p, mem_fid, nm, st);
            DevBuf<int64_t> off;
            DevBuf<int32_t> cl, rk;
            off.reserve(C + 1);
            cl.reserve(ne + 1);
            rk.reserve(ne + 1);
            h2d(off.p, cls_off, C + 1, st);
            h2d(cl.p, cls_id, ne, st);
            h2d(rk.p, cls_rank, ne, st);
            for (int64_t i = 0; i < ne; i++)
                if (cls_id[i] < 0 || cls_id[i] > vocab || cls_rank[i] < 1 || cls_rank[i] > 255)
                    throw Error{FX_E_DATA, "class id / rank outside the encodable range"};
            build_index_from_csr(ix, off.p, cl.p, rk.p, ne, st);
        } catch (...) {
            delete ix;
            throw;
        }
        *out = ix;
    })
}

int fx_index_destroy(fx_index *ix) {
    FX_GUARD({
        if (ix) {
            set_dev(ix->dev);
            cudaStream_t st = ix->st;
            const bool own = ix->owns_stream;
            {
                StreamGuard sg_(st);
                delete ix;
            }
            if (own && st) cudaStreamDestroy(st);
        }
    })
}

int fx_lookup(fx_index *ix, int32_t class_enc, int32_t k_x, int64_t *out_ids, int64_t cap, int64_t *out_n) {
    FX_GUARD({
        if (!ix || !out_n) throw Error{FX_E_USAGE, "null argument"};
        if (k_x < 1 || k_x > ix->K) throw Error{FX_E_KX_TOO_LARGE, "k_x outside [1, K]"};
        *out_n = 0;
        if (class_enc < 0 || class_enc > ix->V) return FX_OK;  // postings.get(c, []) -> []
        set_dev(ix->dev);
        StreamGuard sg_(ix->st);
        *out_n = index_lookup(ix, class_enc, k_x, out_ids, out_ids ? cap : 0);
    })
}

int fx_index_reps(fx_index *ix, int64_t *reps) {
    FX_GUARD({
        if (!ix || !reps) throw Error{FX_E_USAGE, "null argument"};
        set_dev(ix->dev);
        StreamGuard sg_(ix->st);
        if (ix->C) {
            d2h(reps, ix->reps.p, ix->C, ix->st);
            FX_CUDA(cudaStreamSynchronize(ix->st));
        }
    })
}

int fx_session_create(fx_index *ix, const int32_t *rep_label, const int32_t *rep_key, int64_t n_keys,
                      const uint8_t *other_map, fx_session **out) {
    FX_GUARD({
        if (!ix || !out) throw Error{FX_E_USAGE, "null argument"};
        set_dev(ix->dev);
        StreamGuard sg_(ix->st);
        fx_session *ss = new fx_session();
        try {
            ss->ix = ix;
            const int64_t C = ix->C;
            ss->keyed = rep_key != nullptr;
            ss->n_keys = rep_key ? n_keys : C;
            ss->rep_label.reserve(C + 1);
            if (rep_label) h2d(ss->rep_label.p, rep_label, C, ix->st);
            else if (C) k_fill_i32<<<(unsigned)cdiv(C, 256), 256, 0, ix->st>>>(C, -5, ss->rep_label.p);
            if (rep_key) {
                ss->rep_key.reserve(C + 1);
                h2d(ss->rep_key.p, rep_key, C, ix->st);
            }
            ss->memo.reserve((ss->n_keys + 4) & ~3LL);
            FX_CUDA(cudaMemsetAsync(ss->memo.p, 0, (ss->n_keys + 4) & ~3LL, ix->st));
            ss->other_map.reserve(ix->V + 1);
            ss->has_other = other_map != nullptr;
            if (other_map) h2d(ss->other_map.p, other_map, ix->V, ix->st);
            else FX_CUDA(cudaMemsetAsync(ss->other_map.p, 0, ix->V + 1, ix->st));
            session_alloc_bits(ss);
            FX_CUDA(cudaStreamSynchronize(ix->st));
        } catch (...) {
            delete ss;
            throw;
        }
        *out = ss;
    })
}

int fx_session_destroy(fx_session *ss) {
    FX_GUARD({
        if (ss) {
            set_dev(ss->ix->dev);
            StreamGuard sg_(ss->ix->st);
            delete ss;
        }
    })
}

int fx_query(fx_session *ss, int32_t class_enc, int32_t k_x, int32_t mode, int32_t keep_label, int32_t batch_step,
             int32_t has_range, int64_t t0, int64_t t1, fx_query_result *res) {
    FX_GUARD({
        if (!ss || !res) throw Error{FX_E_USAGE, "null argument"};
        fx_index *ix = ss->ix;
        if (class_enc < 0 || class_enc > ix->V) throw Error{FX_E_UNKNOWN_CLASS, "unknown class"};
        int kx = k_x;
        if (mode == 1) kx = (int)ix->K;
        if (kx < 1 || kx > ix->K) throw Error{FX_E_KX_TOO_LARGE, "k_x outside [1, K]"};
        set_dev(ix->dev);
        StreamGuard sg_(ix->st);
        run_query(ss, class_enc, kx, mode, keep_label, batch_step, has_range, t0, t1, res);
    })
}

int fx_query_fetch(fx_session *ss, int64_t *frame_ids, int64_t *object_ids) {
    FX_GUARD({
        if (!ss) throw Error{FX_E_USAGE, "null session"};
        set_dev(ss->ix->dev);
        StreamGuard sg_(ss->ix->st);
        d2h(frame_ids, ss->out_f.p, ss->nf, ss->ix->st);
        d2h(object_ids, ss->out_o.p, ss->no, ss->ix->st);
        FX_CUDA(cudaStreamSynchronize(ss->ix->st));
    })
}

int fx_query_fetch_device(fx_session *ss, int64_t *d_frame_ids, int64_t *d_object_ids) {
    FX_GUARD({
        if (!ss) throw Error{FX_E_USAGE, "null session"};
        set_dev(ss->ix->dev);
        StreamGuard sg_(ss->ix->st);
        cudaStream_t st = ss->ix->st;
        if (ss->nf && d_frame_ids)
            FX_CUDA(cudaMemcpyAsync(d_frame_ids, ss->out_f.p, sizeof(int64_t) * ss->nf, cudaMemcpyDeviceToDevice, st));
        if (ss->no && d_object_ids)
            FX_CUDA(cudaMemcpyAsync(d_object_ids, ss->out_o.p, sizeof(int64_t) * ss->no, cudaMemcpyDeviceToDevice, st));
        FX_CUDA(cudaStreamSynchronize(st));
    })
}

int fx_session_reset(fx_session *ss) {
    FX_GUARD({
        if (!ss) throw Error{FX_E_USAGE, "null session"};
        set_dev(ss->ix->dev);
        StreamGuard sg_(ss->ix->st);
        cudaStream_t st = ss->ix->st;
        FX_CUDA(cudaMemsetAsync(ss->memo.p, 0, (ss->n_keys + 4) & ~3LL, st));
        FX_CUDA(cudaStreamSynchronize(st));
        ss->gt_total = 0;
    })
}

int fx_session_set_labels(fx_session *ss, int64_t n, const int32_t *cluster_idx, const int32_t *labels) {
    FX_GUARD({
        if (!ss || (n > 0 && (!cluster_idx || !labels))) throw Error{FX_E_USAGE, "null argument"};
        set_dev(ss->ix->dev);
        StreamGuard sg_(ss->ix->st);
        session_set_labels(ss, n, cluster_idx, labels);
    })
}

int fx_session_gather_labels(fx_session *ss, const int32_t *labels, int64_t oid_base, int64_t n) {
    FX_GUARD({
        if (!ss || (n > 0 && !labels) || n < 0) throw Error{FX_E_USAGE, "bad argument"};
        set_dev(ss->ix->dev);
        StreamGuard sg_(ss->ix->st);
        session_gather_labels(ss, labels, oid_base, n);
    })
}

int fx_session_needed(fx_session *ss, int32_t *cluster_idx, int64_t *n) {
    FX_GUARD({
        if (!ss || !n) throw Error{FX_E_USAGE, "null argument"};
        *n = ss->n_need;
        if (cluster_idx && ss->n_need) {
            set_dev(ss->ix->dev);
            StreamGuard sg_(ss->ix->st);
            d2h(cluster_idx, ss->need.p, ss->n_need, ss->ix->st);
            FX_CUDA(cudaStreamSynchronize(ss->ix->st));
        }
    })
}

int fx_session_seen_open(fx_session *ss, int32_t *seen_id) {
    FX_GUARD({
        if (!ss || !seen_id) throw Error{FX_E_USAGE, "null argument"};
        set_dev(ss->ix->dev);
        StreamGuard sg_(ss->ix->st);
        auto *b = new DevBuf<uint8_t>();
        try {
            b->reserve(ss->ix->C + 1);
            FX_CUDA(cudaMemsetAsync(b->p, 0, ss->ix->C + 1, ss->ix->st));
            FX_CUDA(cudaStreamSynchronize(ss->ix->st));
        } catch (...) {
            delete b;
            throw;
        }
        size_t i = 0;
        while (i < ss->seen_sets.size() && ss->seen_sets[i]) i++;
        if (i == ss->seen_sets.size()) ss->seen_sets.push_back(b);
        else ss->seen_sets[i] = b;
        *seen_id = (int32_t)i;
    })
}

int fx_session_seen_close(fx_session *ss, int32_t seen_id) {
    FX_GUARD({
        if (!ss) throw Error{FX_E_USAGE, "null session"};
        if (seen_id < 0 || seen_id >= (int32_t)ss->seen_sets.size() || !ss->seen_sets[seen_id])
            throw Error{FX_E_USAGE, "seen set not open"};
        set_dev(ss->ix->dev);
        StreamGuard sg_(ss->ix->st);
        delete ss->seen_sets[seen_id];
        ss->seen_sets[seen_id] = nullptr;
    })
}

int64_t fx_session_gt_total(fx_session *ss) { return ss ? ss->gt_total : 0; }

}  // extern "C"
