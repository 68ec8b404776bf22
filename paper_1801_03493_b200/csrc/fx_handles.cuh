// fx_handles.cuh -- layouts of the opaque C-ABI handles (device-resident state).
#pragma once

#include "fx_internal.cuh"

namespace fx {

// Engine counters (device int64 array `ctr`).
enum Ctr {
    C_NLIVE = 0,       // live clusters
    C_NEXT_CID,        // next cluster id (= clusters created)
    C_DC,              // distance_computations (clustering.py:117)
    C_NFREE,           // free slot stack size
    C_NEVICT_TOTAL,    // clusters evicted so far
    C_EXACT,           // objects resolved through the exact float64 path
    C_NSNAP,           // snapshot live slots of the current batch
    C_NRES,            // residual columns of the current batch
    C_NINSERTED,       // classified objects inserted so far
    C_NEVICT_BATCH,    // evictions in the current batch
    C_NDEFER,          // slots freed in the current batch (reusable next batch)
    C_NOD,             // on-demand in-batch columns of the current batch
    C_LAST_CID,        // cluster of the last classified object (prev_cluster)
    C_NDIRTY,          // slots touched/evicted in the current batch
    C_ERR,             // internal error flag
    C_FAST,            // objects decided by the certain (screen-bounded) path
    C_FCFLAG,          // K1b: objects whose top-K sits within the float64 logit margin
    C_EVCUR,           // eviction cursor: every cid below it is evicted or has size > 1
    C_FASTST,          // resolve fast path of the current batch: 0 not run, 1 committed, 2 fall back
    C_FDONE,           // fast path: CTAs done (last-block election)
    C_FASTB,           // batches committed by the fast path
    C_NOISEFLAG,       // feature noise: exp() decisions within 0.01 ulp of a midpoint (fx_stream_set_feature_noise)
    C_COUNT
};

struct StreamChunkRef {
    // feature rows of classified objects are addressed through frow[cls_idx]
};

}  // namespace fx

struct fx_stream {
    fx_stream_config cfg{};
    int dev = 0;
    cudaStream_t st = nullptr;
    int esize = 4;             // feature element size
    bool tc_screen = false;    // tcgen05 TF32 screen (f32 features, D % 4 == 0)
    bool finalized = false;
    bool debug_check = false;
    bool counted = false;      // included in live_engines(dev)
    bool partitioned = false;  // streams in an SM partition (green context, fx_device_set_partitions)
    bool timing = false;  // per-phase CUDA-event timers (fx_stream_set_timing / FOCUS_B200_TIMERS=1)
    bool rows_aligned16 = true;  // every feature row pointer so far is 16-byte aligned  // FOCUS_B200_CHECK=1: per-batch host-side invariant checks (slow)

    // rank model
    bool has_rm = false;
    int gt = 0;
    uint64_t seed = 0;
    fx::DevBuf<uint64_t> rm_thr;
    fx::DevBuf<int32_t> rm_emit, rm_fill;
    // K1b classifier head
    bool has_fc = false;
    // ingest-time feature noise (fx_stream_set_feature_noise)
    bool has_noise = false;
    double noise_sigma = 0.0;
    uint64_t noise_seed = 0;
    int noise_in_type = 0;
    int fc_V = 0;
    fx::DevBuf<float> fc_W, fc_wnorm, fc_bias;

    // per-object arrays (grow)
    int64_t n_seen = 0, n_cls = 0;
    fx::DevBuf<int64_t> oid, fid;
    fx::DevBuf<uint8_t> is_dup;
    fx::DevBuf<int32_t> topk;       // [n_seen*k]
    fx::DevBuf<int32_t> cluster_of; // [n_seen]
    fx::DevBuf<int32_t> mrank;      // [n_seen] rank in the cluster's member list
    fx::DevBuf<int32_t> frank;      // [n_seen] rank among featured members
    // per-classified arrays
    fx::DevBuf<int64_t> cls_obj;    // [n_cls] object index
    fx::DevBuf<const char *> frow;  // [n_cls] feature row pointer
    fx::DevBuf<float> fnorm;        // [n_cls] ||f|| (fp32, screen error term)
    fx::DevBuf<int32_t> dup_run;    // [n_cls] dups directly following
    std::vector<fx::DevBuf<char> *> owned_feats;  // host-ingested feature copies

    // pixel-diff carry-over
    bool has_prev = false;
    int64_t prev_fid = 0;
    fx::DevBuf<double> prev_sig;

    // clustering engine
    int B = 0;                 // batch size
    int64_t nslots = 0;
    fx::DevBuf<double> S;      // [nslots*D] exact running sums
    fx::DevBuf<float> C32;     // [nslots*D] fp32 centroid snapshot
    fx::DevBuf<int32_t> s_cid, s_nfeat, s_size, s_snapq, s_seedpos, s_foldpos, s_pend, s_odcol, s_didx, s_grp,
        s_evicted, live, live_pos, free_stack, defer_free;
    fx::DevBuf<double> s_drift;
    fx::DevBuf<float> s_cn2;   // ||c||^2 of the snapshot centroid (fp32)
    fx::DevBuf<int64_t> ctr;
    fx::DevBuf<int64_t> prof;  // resolve cycle counters (diagnostics)
    fx::DevBuf<int32_t> snap_slot;  // [nslots]
    // per-batch scratch
    fx::DevBuf<float> dist;    // [B*ld]
    int64_t ld = 0;
    fx::DevBuf<float> dres;    // [B*B]
    fx::DevBuf<int32_t> res_col, res_pos;
    fx::DevBuf<float> dod;     // [B*B] on-demand columns
    fx::DevBuf<int32_t> slot_of, pend_rank, evict_slot, evict_cid, dirty, dirty_off, pend_list, pend_seg, sum_slot, sum_q;
    fx::DevBuf<float> sum_d1, sum_e1, sum_lbr;
    // resolve fast path scratch (k_rfast1 / k_rfast3)
    fx::DevBuf<int32_t> f_rank, f_dup, f_ccnt, f_cdup, f_gi;
    fx::DevBuf<float> f_P, f_csum, f_cmax, f_gf;
    fx::DevBuf<double> f_gd;
    // snapshot tree fold (k_tfold) + lagged exact chain (k_fold on st2)
    fx::DevBuf<double> S_tree;             // [nslots*D] running sums in the tree fold's order
    fx::DevBuf<double> s_abs, s_sdev;      // [nslots] sum of member norms; bound on |snapshot - exact centroid|
    fx::DevBuf<float> tf_cn2;              // [(2B+2) * gx] per-slice ||c||^2 partials
    fx::DevBuf<int32_t> tf_cnt;            // [2B+2] CTAs done per dirty slot (last-block election)
    fx::DevBuf<double> tf_part;            // [TF_SPLIT * D + TF_SPLIT] row-chunk partials of the largest slot
    fx::DevBuf<int32_t> tf_bcnt;           // [gx] row chunks done per column slice
    fx::DevBuf<unsigned char> rs_gobj;     // k_resolve's per-object state when B > 4096 (global instead of smem)
    fx::DevBuf<unsigned long long> chain_epoch;  // [1] lagged chains completed (k_fold's last CTA)
    fx::DevBuf<unsigned int> fold_done;          // [1] k_fold CTAs finished (last-CTA election)
    fx::DevBuf<double> tf_P, tf_PF;        // k_tfold_a piece sums [B * D] (by piece start row), norm sums [B]
    fx::DevBuf<int32_t> cd_meta, cd_off;   // [2][8][2B+3], [2][2B+3] chain descriptors (double buffered)
    fx::DevBuf<const char *> cd_rows;      // [2][B] member rows of the chain (nullptr: already in S)
    fx::DevBuf<int64_t> cd_nd;             // [2] dirty slots of the chain
    cudaStream_t st2 = nullptr;            // the exact float64 chain runs here, one batch behind
    cudaEvent_t ev_tf[2] = {nullptr, nullptr}, ev_ch[2] = {nullptr, nullptr};
    bool chain_pending[2] = {false, false};
    fx::DevBuf<int32_t> rowmin;          // [B+1] multi-tile TC screen: min lower bound per row (float bits)
    fx::DevBuf<float> snorm;             // [ld] snapshot column norms (TC screen)
    const char *abase = nullptr;         // feature rows of the current ingest call (TMA tensor map)
    int64_t arows = 0, a_cbase = 0, a_obj0 = 0;
    bool a_compact = false;
    fx::DevBuf<int32_t> orow;            // [rows of the call] classified index of each object row, -1: duplicate
    fx::DevBuf<float> C32q;              // [ld*D] FP32 snapshot packed in snapshot order (TMA screen)
    fx::DevBuf<int32_t> cid_slot;        // [>= clusters created + 3B] slot of each cluster id
    fx::DevBuf<int32_t> s_fjoin;         // [nslots] first join position inside a window (scratch, INT_MAX)
    fx::DevBuf<int32_t> ev_pos, ev_vic;  // [B+1] window seed positions / eviction victims
    // per-cluster results (grow with clusters)
    int64_t cl_cap = 0;
    fx::DevBuf<double> fcent;      // [cl_cap*D] final centroids
    fx::DevBuf<int32_t> cl_nfeat, cl_size;
    int64_t h_ctr[fx::C_COUNT] = {0};
    int64_t *h_ctr_ring = nullptr;  // pinned [3][C_COUNT], async per-batch readback
    cudaEvent_t ring_ev[3] = {nullptr, nullptr, nullptr};
    int64_t batch_no = 0;

    fx::PwPlan *plan_host = nullptr;
    fx::DevBuf<fx::PwPlan> plan;

    // per-phase device timing (CUDA events, collected at sync points)
    struct Timer {
        cudaEvent_t a = nullptr, b = nullptr;
        int phase = -1;
    };
    std::vector<Timer> timers;  // pool
    std::vector<int> pending;   // indices into timers awaiting collection
    int open_timer = -1;
    double t_ms[16] = {0};  // [0..6] device phases (fx_stream_timings), [8..14] host-side ms per section
    void tstart(int phase);
    void tstop();
    void tcollect();

    ~fx_stream();
};

struct fx_index {
    int dev = 0;
    cudaStream_t st = nullptr;
    bool owns_stream = false;
    int64_t C = 0, D = 0, V = 0, K = 0;
    int64_t n_members = 0, n_cls_entries = 0, n_postings = 0;
    bool has_centroids = false;
    fx::DevBuf<int64_t> cluster_ids;
    fx::DevBuf<double> centroids;
    fx::DevBuf<int64_t> reps;      // representative object id or -1
    fx::DevBuf<int64_t> mem_off, mem_oid, mem_fid;
    fx::DevBuf<int64_t> cls_off;
    fx::DevBuf<int32_t> cls_id, cls_rank;
    fx::DevBuf<int64_t> post_off;  // [V+2]
    fx::DevBuf<int32_t> post_cidx, post_rank;
    std::vector<int64_t> h_post_off;
    int64_t fmin = 0, fmax = -1, omin = 0, omax = -1;
    ~fx_index();
};

struct fx_session {
    fx_index *ix = nullptr;
    int64_t n_keys = 0;
    int64_t gt_total = 0;
    bool has_other = false;
    bool keyed = false;  // rep_key given (else key = cluster index)
    fx::DevBuf<int32_t> rep_label, rep_key;
    fx::DevBuf<uint8_t> memo, other_map;
    fx::DevBuf<uint32_t> fbits, obits;
    fx::DevBuf<int64_t> wprefix_f, wprefix_o;
    fx::DevBuf<int64_t> out_f, out_o;
    fx::DevBuf<int32_t> cand, matched, need;
    fx::DevBuf<int64_t> qctr;
    std::vector<fx::DevBuf<uint8_t> *> seen_sets;  // batched queries (fx_session_seen_open)
    int64_t n_need = 0;
    fx::DevBuf<int64_t> h_pinned_dummy;
    int64_t nf = 0, no = 0;
    ~fx_session();
};
