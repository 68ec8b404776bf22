/*
 * focus_b200.h -- C ABI of the B200-native Focus ingest/query hot path.
 *
 * The drop-in boundary: plain pointers and sizes, no torch
 * types.  Every entry point names the reference (`focusidx`,
 * /root/reference/pkg/src/focusidx) interface it replaces.  A caller binds
 * this with ctypes exactly like the package in
 * paper_1801_03493_b200/ does.
 *
 * Ownership: the library owns all device state behind the opaque handles;
 * callers own every input/output buffer.  Pointers are HOST pointers unless a
 * function says otherwise (the *_device variants take device pointers that
 * must live on the handle's device).
 *
 * Threading: one fx_stream per video stream, single writer
 * (clustering.py:87 "one engine per stream; inserts are strictly
 * sequential").  Different handles may be driven from different host threads
 * and devices.  A built fx_index is immutable and safe for concurrent
 * fx_lookup; an fx_session (like QuerySession._gt_cache, query.py:44) is not.
 *
 * Errors: every function returns an fx_status; the codes map 1:1 onto the
 * reference exception classes (errors.py).  fx_last_error() gives a message.
 */
#ifndef FOCUS_B200_H
#define FOCUS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> focusidx.errors (errors.py:4-95). */
typedef enum {
    FX_OK = 0,
    FX_E_USAGE = 1,                  /* UsageError            errors.py:8-9   */
    FX_E_DATA = 2,                   /* DataError             errors.py:12-13 */
    FX_E_VALUE = 3,                  /* ValueError: bad number literal in a stream file (streamio.py:91-95) */
    FX_E_UNKNOWN_PROFILE = 10,       /* UnknownProfile        errors.py:18-19 */
    FX_E_K_OUT_OF_RANGE = 11,        /* KOutOfRange           errors.py:22-23 */
    FX_E_NON_POSITIVE_M = 12,        /* NonPositiveM          errors.py:26-27 */
    FX_E_MISSING_TRUE_CLASS = 20,    /* MissingTrueClass      errors.py:32-33 */
    FX_E_DIMENSION_MISMATCH = 30,    /* DimensionMismatch     errors.py:42-43 */
    FX_E_SIGNATURE_LENGTH = 31,      /* SignatureLengthMismatch errors.py:46-47 */
    FX_E_DUPLICATE_CLUSTER_ID = 40,  /* DuplicateClusterId    errors.py:52-53 */
    FX_E_FORMAT_VERSION = 41,        /* FormatVersionMismatch errors.py:56-57 */
    FX_E_CHECKSUM = 42,              /* ChecksumMismatch      errors.py:60-61 */
    FX_E_KX_TOO_LARGE = 50,          /* KxTooLarge            errors.py:66-67 */
    FX_E_UNKNOWN_CLASS = 51,         /* UnknownClass          errors.py:70-71 */
    FX_E_NON_MONOTONE_SCHEDULE = 52, /* NonMonotoneSchedule   errors.py:74-75 */
    FX_E_MISSING_OBJECT = 60,        /* KeyError: objects[rep] absent (query.py:58) */
    FX_E_NEED_LABELS = 70,           /* not an error: fx_query needs GT labels of some
                                        representatives first (fx_session_needed) */
    FX_E_CUDA = 90,                  /* CUDA runtime / launch failure */
    FX_E_OOM = 91,                   /* device allocation failed */
    FX_E_INTERNAL = 99
} fx_status;

/* Feature element type accepted by fx_ingest (DetectedObject.feature,
 * core.py:37-50; the reference upcasts to float64 everywhere). */
enum { FX_F32 = 0, FX_F64 = 1 };

/* Class encoding on the wire: 0..V-1 real classes, V = OTHER_CLASS
 * (core.py:18, 24-34). */

/* ------------------------------------------------------------------------ */
/* Stream engine: replaces ingest.ingest_stream's loop + ClusterEngine       */
/* (ingest.py:50-96, clustering.py:86-160).                                  */
/* ------------------------------------------------------------------------ */

typedef struct fx_stream fx_stream;

typedef struct {
    int32_t dim;       /* header.dim: feature dimension D               */
    int32_t sig_dim;   /* header.sig_dim: pixel signature length S      */
    int32_t vocab;     /* header.vocab: V                               */
    int32_t k;         /* cfg.k: classes indexed per object             */
    double t;          /* cfg.t: L2 join threshold T (inclusive)        */
    int64_t m;         /* cfg.m: cap on live clusters                   */
    double pixel_eps;  /* ingest pixel_eps (negative disables)          */
    int32_t feat_type; /* FX_F32 or FX_F64                              */
    int32_t device;    /* CUDA device ordinal                           */
    int32_t batch;     /* objects per clustering batch, 0 = auto        */
    int32_t partition; /* SM partition (fx_device_set_partitions): p > 0
                          = partition p-1, 0 = next in round-robin order */
} fx_stream_config;

/* Device rank model (the synthetic "cheap CNN" top-K, classifiers.py:59-70,
 * 110-149).  The host derives these tables from the ClassifierProfile:
 *   thresholds[j], j = 0..k-1: smallest 53-bit uniform integer u (the
 *     draw is u * 2^-53, first Generator.random() of
 *     default_rng([seed, object_id, 0])) whose rank_from_uniform is >= j+2;
 *     UINT64_MAX when unreachable.  Rank 1 below thresholds[0].
 *   emit_map[c], c = 0..V-1: profile.map_class(c) encoded (OTHER = V).
 *   fillers[e*k + j]: _confusion_order(..., emitted=e)[j], encoded, for every
 *     emitted class e in 0..V.                                              */
typedef struct {
    int32_t ground_truth; /* kind == GROUND_TRUTH: rank is always 1 */
    int32_t reserved;
    uint64_t seed;        /* ingest seed (rng_seed) */
    const uint64_t *thresholds;
    const int32_t *emit_map;
    const int32_t *fillers;
} fx_rank_model;

int fx_stream_create(const fx_stream_config *cfg, fx_stream **out);
int fx_stream_destroy(fx_stream *s);
int fx_stream_set_rank_model(fx_stream *s, const fx_rank_model *rm);

/* K1b cheap-CNN classifier head (north star kernel 1; no reference function:
 * it is what a classify_fn plugged into ingest.py:52-61,73 computes):
 * logits = feature . W^T + bias over `vocab` classes, top-k by descending
 * logit (ties -> smaller class id).  W: vocab x dim float32 row-major, bias:
 * vocab float32 or NULL (host pointers, copied).  Once set, fx_ingest needs
 * neither true_class nor topk; FP32 features, dim % 4 == 0, k <= 16. */
int fx_stream_set_fc_head(fx_stream *s, int32_t vocab, const float *W, const float *bias);

/* K1b standalone over n dense float32 feature rows (host pointers):
 * out_topk[n*k] classes, out_conf[n*k] softmax confidences (may be NULL),
 * out_flag[n] 1 where float64 logits among ranks 1..k+1 are within their
 * error bound of each other (may be NULL). */
int fx_fc_topk(int32_t device, int64_t n, int32_t dim, int32_t vocab, int32_t k, const float *feats, const float *W,
               const float *bias, int32_t *out_topk, float *out_conf, uint8_t *out_flag);
/* Same with DEVICE pointers, enqueued on the caller's CUDA stream
 * (cudaStream_t passed as void*; NULL = legacy default stream); returns after
 * enqueueing (scratch is stream-ordered). */
int fx_fc_topk_device(int32_t device, void *cuda_stream, int64_t n, int32_t dim, int32_t vocab, int32_t k,
                      const float *d_feats, const float *d_W, const float *d_bias, int32_t *d_topk, float *d_conf,
                      uint8_t *d_flag);

/* extract_feature (classifiers.py:152-158) on the device, bit for bit:
 * out[i] = feats[i] + sigma * default_rng([seed, object_ids[i], 1]).standard_normal(dim)
 * (numpy SeedSequence + PCG64 + ziggurat; float64 arithmetic, as numpy
 * promotes feature + float64 noise).  sigma == 0 copies the features (the
 * reference's early return).  feats[n*dim] of feat_type (FX_F32 / FX_F64),
 * out[n*dim] float64.  *n_flagged (may be NULL): u-layer rejection tests
 * whose exp() sat within 0.01 ulp of a rounding midpoint (expected 0).
 * Replaces the per-object numpy call at classifiers.py:156-158. */
int fx_extract_features(int32_t device, int64_t n, int32_t dim, const int64_t *object_ids, const void *feats,
                        int32_t feat_type, double sigma, uint64_t seed, double *out, int64_t *n_flagged);
/* Same with DEVICE pointers and row strides (elements), enqueued on the
 * caller's CUDA stream (void*, NULL = legacy default stream);
 * d_flagged: device uint64 counter incremented (may be NULL). */
int fx_extract_features_device(int32_t device, int64_t n, int32_t dim, const int64_t *d_object_ids,
                               const void *d_feats, int32_t feat_type, int64_t ld_in, double sigma, uint64_t seed,
                               double *d_out, int64_t ld_out, uint64_t *d_flagged, void *cuda_stream);
/* Ingest-time feature noise (the drop-in ingest_stream with the synthetic
 * classifier profile, classifiers.py:152-158): fx_ingest's feature rows are
 * the objects' RAW features (of in_type, FX_FEATS_COMPACT rows of the
 * classified objects) and the engine clusters extract_feature of them,
 * computed on the device.  The stream's feat_type must be FX_F64 when
 * sigma > 0 (numpy's result type).  Host-buffer fx_ingest only. */
int fx_stream_set_feature_noise(fx_stream *s, double sigma, uint64_t seed, int32_t in_type);

/* pixel_diff (ingest.py:37-47) of every object against its predecessor in
 * a sequence, without an engine: out_is_dup[0] = 0, out_is_dup[i] =
 * pixel_diff(obj[i-1], obj[i], eps).  sigs[n * sig_dim] float64. */
int fx_dup_flags(int32_t device, int64_t n, int32_t sig_dim, const int64_t *frame_ids, const double *sigs,
                 double eps, uint8_t *out_is_dup);

/* pixel_diff over a chunk (ingest.py:37-47), continuing from the previous
 * chunk's last object; does not consume the chunk.  out_is_dup[n]. */
int fx_stream_dup_flags(fx_stream *s, int64_t n, const int64_t *frame_ids, const double *sigs,
                        uint8_t *out_is_dup);

/* Ingest the next chunk of n objects in stream order (object ids strictly
 * increasing).  Either true_class (rank model; -2 = unlabeled) or topk
 * (n x k encoded classes from an external classify_fn; rows of duplicates
 * ignored) must be given.  feats: n x dim of cfg.feat_type; if
 * FX_FEATS_COMPACT is set it holds only the rows of non-duplicate objects.
 * Host pointers. */
enum { FX_FEATS_COMPACT = 1 };
int fx_ingest(fx_stream *s, int64_t n, const int64_t *object_ids, const int64_t *frame_ids,
              const double *sigs, const void *feats, const int32_t *true_class,
              const int32_t *topk, int32_t flags);
/* fx_ingest with FX_FEATS_COMPACT host rows whose count the caller knows
 * (n_feat_rows = classified objects): the feature rows start crossing PCIe
 * immediately, in chunks, while pixel differencing places the object chunks
 * (the e2e path: nothing waits for K0 before the big copy starts).
 * FX_E_USAGE if n_feat_rows differs from the classified objects K0 finds. */
int fx_ingest_rows(fx_stream *s, int64_t n, const int64_t *object_ids, const int64_t *frame_ids, const double *sigs,
                   const void *feats, int64_t n_feat_rows, const int32_t *true_class, const int32_t *topk);
/* Same with device pointers (inputs already resident in HBM). */
int fx_ingest_device(fx_stream *s, int64_t n, const int64_t *object_ids, const int64_t *frame_ids,
                     const double *sigs, const void *feats, const int32_t *true_class,
                     const int32_t *topk, int32_t flags);

/* IngestReport (ingest.py:26-34) minus the float cost fields (the host
 * multiplies by profile.cost_units). */
typedef struct {
    int64_t objects_seen;
    int64_t objects_classified;
    int64_t clusters_emitted;
    int64_t distance_computations;
    int64_t gt_invocations; /* always 0 */
    int64_t exact_rechecks; /* objects resolved by the exact float64 path */
} fx_ingest_report;

/* Seal everything, build the top-K index on the device (finalize,
 * clustering.py:146-153 + index.build, index.py:60-72).  The stream handle
 * stays valid for fx_stream_* queries but accepts no more objects. */
typedef struct fx_index fx_index;
int fx_finalize(fx_stream *s, fx_index **out, fx_ingest_report *report);

/* Per-object results of the ingest (n_seen entries, stream order). */
int fx_stream_object_results(fx_stream *s, int32_t *cluster_of, uint8_t *is_dup, int32_t *topk);

/* ------------------------------------------------------------------------ */
/* Index: TopKIndex (index.py:50-85)                                          */
/* ------------------------------------------------------------------------ */

typedef struct {
    int64_t n_clusters;
    int64_t dim;
    int64_t n_members;      /* sum of cluster sizes (incl. dedup members) */
    int64_t n_class_entries;/* sum of |class_best_rank| */
    int64_t n_postings;     /* sum of |postings[c]| over classes */
    int64_t vocab;
    int64_t k;
    int64_t has_centroids;
} fx_index_sizes;

int fx_index_sizes_get(fx_index *ix, fx_index_sizes *out);

/* Copy the index out (any pointer may be NULL to skip).  Cluster ids are
 * 0..n_clusters-1 for ingested indexes.
 *   cluster_ids[C], centroids[C*dim] (float64), reps[C] (-1 = None),
 *   mem_off[C+1], mem_oid[n_members], mem_fid[n_members],
 *   cls_off[C+1], cls_id[n_class_entries] (encoded, ascending per cluster),
 *   cls_rank[n_class_entries],
 *   post_off[V+2] (class c in [post_off[c], post_off[c+1])),
 *   post_cluster[n_postings] (ascending per class). */
int fx_index_export(fx_index *ix, int64_t *cluster_ids, double *centroids, int64_t *reps,
                    int64_t *mem_off, int64_t *mem_oid, int64_t *mem_fid, int64_t *cls_off,
                    int32_t *cls_id, int32_t *cls_rank, int64_t *post_off, int64_t *post_cluster);

/* index.build from caller-provided cluster records (index.py:60-72): the
 * postings are built on the device.  Cluster ids may be arbitrary int64 and
 * in any order; FX_E_DUPLICATE_CLUSTER_ID on repeats.  CSR layout as in
 * fx_index_export.  centroids may be NULL. */
int fx_index_build(int64_t n_clusters, int32_t vocab, int32_t k, int32_t dim, int32_t device,
                   const int64_t *cluster_ids, const double *centroids, const int64_t *reps,
                   const int64_t *mem_off, const int64_t *mem_oid, const int64_t *mem_fid,
                   const int64_t *cls_off, const int32_t *cls_id, const int32_t *cls_rank,
                   fx_index **out);
int fx_index_destroy(fx_index *ix);

/* index.save (index.py:88-131, FOCUSIDX/1): writes to `path` exactly the
 * bytes of the reference's _render -- `head` (magic, stream_id=, D=, V=, n=,
 * config lines and "[CLUSTERS]\n", built by the caller), one line per
 * cluster in id order (centroid %.9g, members, frames, class:rank by encoded
 * class), "[POSTINGS]", the non-empty postings by encoded class and the
 * CRC32 trailer.  Arrays in the fx_index_export layout (host memory;
 * centroids required).  Host-only: runs without a GPU.  threads <= 0: all
 * hardware threads. */
/* streamio.read_stream (streamio.py:58-113), FOCUSSTREAM/1, decoded by host
 * threads.  open: reads the file, checks magic and header, indexes the
 * object lines (FX_E_FORMAT_VERSION, FX_E_DATA).  header: stream_id (NUL-
 * terminated, cap bytes), fps, D, S, V, object count.  read: parses every
 * object line into caller arrays -- object/frame ids, true class (decoded:
 * OTHER = -1, unlabeled = -2), signatures (n x S float64), features (n x D,
 * float32 if feats_f32 else float64); the first bad line in file order
 * raises what the reference raises (FX_E_DATA, FX_E_VALUE).  Host-only. */
typedef struct fx_stream_file fx_stream_file;
int fx_stream_file_open(const char *path, fx_stream_file **out);
int fx_stream_file_header(fx_stream_file *f, char *stream_id, int64_t cap, double *fps, int32_t *dim,
                          int32_t *sig_dim, int32_t *vocab, int64_t *n_objects);
int fx_stream_file_read(fx_stream_file *f, int64_t *object_ids, int64_t *frame_ids, int32_t *true_class,
                        double *sigs, void *feats, int32_t feats_f32, int32_t threads);
int fx_stream_file_close(fx_stream_file *f);

int fx_index_write(const char *path, const char *head, int64_t head_len, int64_t n_clusters, int32_t dim,
                   int32_t vocab, const int64_t *cluster_ids, const double *centroids, const int64_t *reps,
                   const int64_t *mem_off, const int64_t *mem_oid, const int64_t *mem_fid,
                   const int64_t *cls_off, const int32_t *cls_id, const int32_t *cls_rank,
                   const int64_t *post_off, const int64_t *post_cluster, int32_t threads);

/* FOCUSIDX/1 reader: index.load (index.py:131-204).  Host-only.
 * fx_index_read: read + newline translation + CRC-32 trailer + magic + the
 *   [CLUSTERS] marker (ChecksumMismatch / FormatVersionMismatch / DataError;
 *   ValueError for a file that is not utf-8);
 * fx_index_file_header: the header lines ('\n'-joined) for the caller to
 *   parse (IndexHeader, Config) -- their errors come first in the reference;
 * fx_index_file_parse(V): cluster records and postings, the reference's
 *   first error in its evaluation order (DataError, DuplicateClusterId,
 *   ValueError);
 * fx_index_file_sizes: [clusters, centroid values, members, frames, class
 *   entries, posting classes, posting ids];
 * fx_index_file_export: file-order CSR arrays (classes decoded: OTHER = -1;
 *   cmid = INT64_MIN for an empty representative field). */
typedef struct fx_index_file fx_index_file;
int fx_index_read(const char *path, fx_index_file **out);
int fx_index_file_header(const fx_index_file *f, char *buf, int64_t cap, int64_t *len);
int fx_index_file_parse(fx_index_file *f, int64_t vocab);
int fx_index_file_sizes(const fx_index_file *f, int64_t *out);
int fx_index_file_export(const fx_index_file *f, int64_t *cid, int64_t *cmid, int64_t *cen_off, double *cen,
                         int64_t *mem_off, int64_t *mem, int64_t *fr_off, int64_t *fr, int64_t *cls_off,
                         int32_t *cls, int32_t *rank, int32_t *post_cls, int64_t *post_off, int64_t *post_ids);
int fx_index_file_free(fx_index_file *f);

/* index.lookup (index.py:75-85): cluster ids posted under class_enc with
 * best rank <= k_x (k_x <= 0 -> K), ascending.  Two-call sizing: pass
 * out_ids = NULL to get *out_n. */
int fx_lookup(fx_index *ix, int32_t class_enc, int32_t k_x, int64_t *out_ids, int64_t cap,
              int64_t *out_n);

/* ------------------------------------------------------------------------ */
/* Query session: QuerySession (query.py:36-154)                             */
/* ------------------------------------------------------------------------ */

typedef struct fx_session fx_session;

/* rep_label[C] (in cluster-index order of the index): ground_truth_label of
 * each cluster's representative (classifiers.py:161-165), or
 *   -2 = representative object has no true class (MissingTrueClass on touch),
 *   -3 = representative object missing from `objects` (KeyError on touch),
 *   -4 = cluster has no representative,
 *   -5 = not known yet: fx_query returns FX_E_NEED_LABELS when a candidate
 *        has it (labels are produced lazily, like _verify, query.py:53-60).
 *   rep_label == NULL: every label starts at -5.
 * rep_key[C]: memo key per cluster (equal keys share one GT inference, the
 *   session memo is keyed by representative object id, query.py:53-60);
 *   keys are dense 0..n_keys-1.  rep_key == NULL: key = cluster index
 *   (representatives of distinct clusters are distinct objects).
 * other_map[V] (may be NULL): 1 if ingest_profile.map_class(c) == OTHER;
 *   labels outside [0, V) map to OTHER (classifiers.py:103-107). */
int fx_session_create(fx_index *ix, const int32_t *rep_label, const int32_t *rep_key,
                      int64_t n_keys, const uint8_t *other_map, fx_session **out);
/* Set labels of n clusters (cluster indexes, host arrays). */
int fx_session_set_labels(fx_session *ss, int64_t n, const int32_t *cluster_idx, const int32_t *labels);
/* Labels from a dense host table indexed by object id - oid_base
 * (labels[i] = GT label of object oid_base + i, -2 = unlabeled); gathered
 * for every representative on the device (reps outside the table -> -3). */
int fx_session_gather_labels(fx_session *ss, const int32_t *labels, int64_t oid_base, int64_t n);
/* After FX_E_NEED_LABELS: *n = number of candidate clusters whose label is
 * unknown; cluster_idx (may be NULL) receives them. */
int fx_session_needed(fx_session *ss, int32_t *cluster_idx, int64_t *n);
/* Representative object id per cluster index (-1 = none), host array [C]. */
int fx_index_reps(fx_index *ix, int64_t *reps);
/* A seen set for one batched_query (query.py:139-154): each generator owns
 * one, so interleaved generators do not share state. */
int fx_session_seen_open(fx_session *ss, int32_t *seen_id);
int fx_session_seen_close(fx_session *ss, int32_t seen_id);
int fx_session_destroy(fx_session *ss);

typedef struct {
    int64_t n_frames;
    int64_t n_objects;
    int64_t gt_inferences;
    int64_t clusters_examined;
    int64_t clusters_matched;
    int64_t error_cluster; /* cluster index that raised, or -1 */
} fx_query_result;

/* One verified query (query.py:75-114):
 *   mode 0: plain execute_query(class_enc, k_x, range);
 *   mode 1: keep_label path of query_other (OTHER postings, k_x = K,
 *           keep clusters whose GT label == keep_label);
 *   batch_step: 0 = independent query; s > 0 = a step of the batched
 *           query whose seen set is fx_session_seen_open's id s - 1 (skip
 *           clusters in it, then add the candidates to it).
 * has_range/t0/t1: inclusive frame range filter.  Results stay in the
 * session until fx_query_fetch. */
int fx_query(fx_session *ss, int32_t class_enc, int32_t k_x, int32_t mode, int32_t keep_label,
             int32_t batch_step, int32_t has_range, int64_t t0, int64_t t1, fx_query_result *res);
int fx_query_fetch(fx_session *ss, int64_t *frame_ids, int64_t *object_ids);
/* Same into DEVICE buffers on the index's device (stream-ordered copy on the
 * index's CUDA stream, completed before return) -- the sharded query merge
 * all-gathers these over NCCL without a host round trip. */
int fx_query_fetch_device(fx_session *ss, int64_t *d_frame_ids, int64_t *d_object_ids);
/* Forget every verification of the session (memo, batched-query seen set,
 * gt total): a fresh QuerySession over the same index (query.py:36-48). */
int fx_session_reset(fx_session *ss);
int64_t fx_session_gt_total(fx_session *ss);

/* ------------------------------------------------------------------------ */
/* Tuner grid evaluation: _GridEvaluator._positions (tuner.py:243-256)         */
/* ------------------------------------------------------------------------ */

/* 0-based position of each queried class in every object's full ranked
 * output of one profile (classify(...).classes(), classifiers.py:136-149):
 * rank from the object's SeedSequence/PCG64 draw (seed, oid, 0) and the
 * profile's rank thresholds (n_thr = output length - 1; ground_truth: rank
 * 1), then the class's index in the emitted class's confusion order --
 * inv[e * v1 + c] (classes encoded, OTHER = V; -1 = absent -> position 0).
 * emitted[n]: the profile's emitted class of each object's true class.
 * out_pos[n_classes * n], class-major.  Host buffers. */
int fx_rank_positions(int32_t device, int64_t n, const int64_t *oids, const int32_t *emitted, uint64_t seed,
                      int32_t ground_truth, int32_t n_thr, const uint64_t *thresholds, const int32_t *inv,
                      int32_t v1, int32_t n_classes, const int32_t *classes, int32_t *out_pos);

/* ------------------------------------------------------------------------ */
/* Misc                                                                       */
/* ------------------------------------------------------------------------ */

const char *fx_last_error(void);
int fx_version(void);

/* SM partitions for several engines on one device: engines created after this
 * call run their streams in SM partition (i mod n_groups) -- CUDA green
 * contexts of ~SMs/n_groups SMs each -- so concurrent engines cannot starve
 * each other's CTAs.  n_groups <= 1 turns it off for engines created later.
 * *out_sms_per_group (may be NULL): SMs per partition.  The reference has no
 * counterpart (its cross-stream parallelism is process-level). */
int fx_device_set_partitions(int32_t device, int32_t n_groups, int32_t *out_sms_per_group);
/* Number of this library's kernels launched so far (process-wide). */
int64_t fx_kernel_launches(void);
/* Device time (CUDA events on the stream's CUDA stream) accumulated over all
 * fx_ingest / fx_finalize calls on s, in ms per phase:
 * out[0] K0+K1a (dup flags, compaction, rank top-K), out[1] K2 screen,
 * out[2] K2 resolve, out[3] K2 fold, out[4] seal, out[5] index build (K3),
 * out[6] number of clustering batches. */
int fx_stream_timings(fx_stream *s, double *out, int n);
/* Per-phase timers are off by default (their events sit between kernels);
 * on = 1 records them for every later batch (also FOCUS_B200_TIMERS=1). */
int fx_stream_set_timing(fx_stream *s, int32_t on);
/* Engine counters: live, clusters, distance_computations, ... (see
 * fx_handles.cuh Ctr); out[i] for i < n. */
int fx_stream_counters(fx_stream *s, int64_t *out, int n);
/* The cudaStream_t the stream's kernels run on (for caller-side CUDA events). */
void *fx_stream_cuda_stream(fx_stream *s);

/* Diagnostic: run the tcgen05 TF32 screen kernel on host matrices
 * A[na x dim], B[nb x dim] (float32, dim % 4 == 0); out[na x nb] receives
 * ||a||^2 + ||b||^2 - 2 a.b as the ingest screen computes it. */
int fx_debug_screen_tc(int32_t device, int64_t na, int64_t nb, int32_t dim, const float *A, const float *B,
                       float *out);

#ifdef __cplusplus
}
#endif
#endif /* FOCUS_B200_H */
