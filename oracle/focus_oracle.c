/*
 * focus_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference `focusidx` ingest hot path
 * (/root/reference/pkg/src/focusidx), used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg.  Nothing in
 * paper_1801_03493_b200/ links or calls this file.
 *
 * Every function cites the reference line it restates.  Third-party
 * arithmetic the reference relies on (numpy 2.3.5, the effective version in
 * this image; pyproject pins only numpy>=1.24) is restated from its published
 * algorithm:
 *   - numpy pairwise summation (add.reduce over a contiguous float64 row),
 *     used by np.linalg.norm(axis=1) and np.mean;
 *   - numpy SeedSequence (pool size 4) + PCG64 (XSL-RR 128/64) + random().
 * Parity is pinned against golden vectors produced by the reference itself
 * (tools/gen_golden.py -> tests/golden/) and, for the numpy primitives,
 * against numpy directly (tests/test_oracle.py).
 *
 * Build: make -C oracle   (gcc -O2 -ffp-contract=off: no FMA contraction,
 * IEEE round-to-nearest everywhere, glibc log() exactly as CPython math.log).
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* numpy pairwise summation                                                  */
/* ------------------------------------------------------------------------ */

/* numpy/_core/src/umath/loops_utils.h.src: pairwise_sum (PW_BLOCKSIZE=128). */
static double pw_sum_block(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum_block(a, n2) + pw_sum_block(a + n2, n - n2);
    }
}

/* pw_sum_block over x[i] = (c[i] - f[i])^2 without materialising x: the same
 * operations in the same order (bit-identical), fused for the distance rows. */
static double pw_sqdiff_block(const double *c, const double *f, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) {
            const double x = c[i] - f[i];
            res += x * x;
        }
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) {
            const double x = c[j] - f[j];
            r[j] = x * x;
        }
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) {
                const double x = c[i + j] - f[i + j];
                r[j] += x * x;
            }
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) {
            const double x = c[i] - f[i];
            res += x * x;
        }
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sqdiff_block(c, f, n2) + pw_sqdiff_block(c + n2, f + n2, n - n2);
    }
}

/* add.reduce of a contiguous float64 row: identity 0.0 plus one pairwise sum
 * over the whole row (verified against numpy 2.3.5 up to n = 70001 in
 * tests/test_oracle.py; the ufunc hands a contiguous unbuffered row over in
 * one inner-loop call). */
ORC_API double orc_pairwise_sum(const double *a, int64_t n) { return 0.0 + pw_sum_block(a, n); }

/* ------------------------------------------------------------------------ */
/* numpy SeedSequence + PCG64                                                */
/* ------------------------------------------------------------------------ */

#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

typedef unsigned __int128 u128;

static uint32_t ss_hashmix(uint32_t v, uint32_t *hc) {
    v ^= *hc;
    *hc *= SS_MULT_A;
    v *= *hc;
    v ^= v >> 16;
    return v;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

/* numpy/random/bit_generator.pyx: SeedSequence.mix_entropy + generate_state(4, uint64)
 * for entropy = the little-endian uint32 words of each (non-negative) int. */
static void ss_state4(const uint64_t *ints, int nints, uint64_t out[4]) {
    uint32_t ent[64];
    int ne = 0;
    for (int i = 0; i < nints; i++) {
        uint64_t v = ints[i];
        if (v == 0) {
            ent[ne++] = 0;
        } else {
            while (v) {
                ent[ne++] = (uint32_t)(v & 0xffffffffu);
                v >>= 32;
            }
        }
    }
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < ne ? ent[i] : 0u, &hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    for (int s = 4; s < ne; s++)
        for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
    uint32_t hb = SS_INIT_B;
    uint32_t w[8];
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    for (int i = 0; i < 4; i++) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

typedef struct {
    u128 state, inc;
} pcg64_t;

static const u128 PCG_MULT = (((u128)0x2360ed051fc65da4ull) << 64) | 0x4385df649fccf645ull;

static void pcg_step(pcg64_t *g) { g->state = g->state * PCG_MULT + g->inc; }

/* numpy pcg64.c: pcg64_set_seed(seed=w[0..1], inc=w[2..3]) -> srandom_r. */
static void pcg_seed(pcg64_t *g, const uint64_t w[4]) {
    u128 initstate = (((u128)w[0]) << 64) | w[1];
    u128 initseq = (((u128)w[2]) << 64) | w[3];
    g->state = 0;
    g->inc = (initseq << 1) | 1u;
    pcg_step(g);
    g->state += initstate;
    pcg_step(g);
}

static uint64_t pcg_next64(pcg64_t *g) {
    pcg_step(g);
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(g->state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

/* First Generator.random() of np.random.default_rng([a, b, c]):
 * classifiers.py:132-133 (rank draw, c=0) and :157 (noise stream, c=1). */
ORC_API double orc_first_uniform3(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t ints[3] = {a, b, c}, w[4];
    ss_state4(ints, 3, w);
    pcg64_t g;
    pcg_seed(&g, w);
    return (double)(pcg_next64(&g) >> 11) * (1.0 / 9007199254740992.0);
}

/* Raw first uint64 of default_rng(ints) -- exposed for primitive tests. */
ORC_API uint64_t orc_first_u64(const uint64_t *ints, int nints) {
    uint64_t w[4];
    ss_state4(ints, nints, w);
    pcg64_t g;
    pcg_seed(&g, w);
    return pcg_next64(&g);
}

/* ------------------------------------------------------------------------ */
/* rank model (classifiers.py:59-70, 126-133)                                */
/* ------------------------------------------------------------------------ */

ORC_API int64_t orc_rank_from_uniform(double u, double p1, double rho, int64_t out_len) {
    if (u <= p1 || out_len == 1) return 1;
    if (rho == 0.0) return out_len < 2 ? out_len : 2;
    double q = log((1.0 - u) / (1.0 - p1)) / log(rho);
    int64_t k = 2 + (int64_t)floor(q);
    if (k < 2) k = 2;
    return k < out_len ? k : out_len;
}

/* true_class_rank for every object: GT profile -> 1, else rank of the first
 * uniform of default_rng([seed, oid, 0]).  has_label[i]==0 -> rank -1 (the
 * caller raises MissingTrueClass, classifiers.py:128-129). */
ORC_API void orc_ranks(int64_t n, uint64_t seed, const int64_t *oids, const uint8_t *has_label,
                       int is_gt, double p1, double rho, int64_t out_len, int32_t *out_rank) {
    for (int64_t i = 0; i < n; i++) {
        if (!has_label[i]) {
            out_rank[i] = -1;
            continue;
        }
        if (is_gt) {
            out_rank[i] = 1;
            continue;
        }
        double u = orc_first_uniform3(seed, (uint64_t)oids[i], 0);
        out_rank[i] = (int32_t)orc_rank_from_uniform(u, p1, rho, out_len);
    }
}

/* ------------------------------------------------------------------------ */
/* pixel differencing (ingest.py:37-47, 69-71)                               */
/* ------------------------------------------------------------------------ */

/* mean |prev - cur| over S signature values, numpy np.mean semantics. */
static double sig_mad(const double *a, const double *b, int s, double *tmp) {
    for (int j = 0; j < s; j++) tmp[j] = fabs(a[j] - b[j]);
    return orc_pairwise_sum(tmp, s) / (double)s;
}

/* is_dup[i] = (i>0) && pixel_diff(obj[i-1], obj[i], eps). Object 0 never dup. */
ORC_API void orc_dup_flags(int64_t n, int s, const int64_t *fids, const double *sigs, double eps,
                           uint8_t *is_dup) {
    double *tmp = (double *)malloc(sizeof(double) * (s > 0 ? s : 1));
    for (int64_t i = 0; i < n; i++) {
        is_dup[i] = 0;
        if (i == 0 || eps < 0) continue;
        if (fids[i] - fids[i - 1] > 1) continue;
        is_dup[i] = sig_mad(sigs + (i - 1) * s, sigs + i * s, s, tmp) <= eps;
    }
    free(tmp);
}

/* ------------------------------------------------------------------------ */
/* ClusterEngine (clustering.py:86-160)                                      */
/* ------------------------------------------------------------------------ */

typedef struct {
    int64_t *v;
    int64_t n, cap;
} vec_i64;

static void vpush(vec_i64 *a, int64_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? a->cap * 2 : 4;
        a->v = (int64_t *)realloc(a->v, sizeof(int64_t) * a->cap);
    }
    a->v[a->n++] = x;
}

typedef struct {
    double *v;
    int64_t n, cap;
} vec_f64;

static void fpush(vec_f64 *a, double x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? a->cap * 2 : 4;
        a->v = (double *)realloc(a->v, sizeof(double) * a->cap);
    }
    a->v[a->n++] = x;
}

typedef struct {
    double *sum;      /* _feature_sum (freed at seal) */
    double *centroid; /* current / final centroid */
    vec_i64 members, frames, featured; /* featured: row index into the feature array */
    vec_i64 featured_oid;
    vec_f64 ins_dist;
    vec_i64 cls_rank; /* pairs (class, best rank), dict insertion order */
    int64_t rep;      /* centroid_member_id, -1 = None */
    int sealed;
} orc_cluster;

typedef struct {
    int dim;
    double t;
    int64_t m;
    const double *feats; /* caller-owned n x dim float64 features */
    orc_cluster *cl;
    int64_t ncl, capcl;
    int64_t *live; /* ascending cluster ids */
    int64_t nlive, caplive;
    int64_t distance_computations;
    int64_t margin_t, margin_tie; /* objects within MARGIN_REL of T / of a tie */
    double *dbuf, *diff, *tdiff;
    int64_t dbuf_cap;
    int nthreads;
} orc_engine;

static int g_threads = 1;
/* threads used for the per-insert distance row (bench's reference arm) */
ORC_API void orc_set_threads(int n) { g_threads = n > 0 ? n : 1; }
ORC_API int orc_get_threads(void) { return g_threads; }

ORC_API orc_engine *orc_engine_new(int dim, double t, int64_t m, const double *feats) {
    orc_engine *e = (orc_engine *)calloc(1, sizeof(orc_engine));
    e->dim = dim;
    e->t = t;
    e->m = m;
    e->feats = feats;
    e->diff = (double *)malloc(sizeof(double) * (dim > 0 ? dim : 1));
    e->nthreads = g_threads;
    e->tdiff = (double *)malloc(sizeof(double) * (dim > 0 ? dim : 1) * (size_t)e->nthreads);
    return e;
}

ORC_API void orc_engine_free(orc_engine *e) {
    if (!e) return;
    for (int64_t i = 0; i < e->ncl; i++) {
        orc_cluster *c = &e->cl[i];
        free(c->sum);
        free(c->centroid);
        free(c->members.v);
        free(c->frames.v);
        free(c->featured.v);
        free(c->featured_oid.v);
        free(c->ins_dist.v);
        free(c->cls_rank.v);
    }
    free(e->cl);
    free(e->live);
    free(e->dbuf);
    free(e->diff);
    free(e->tdiff);
    free(e);
}

/* ||c - f||_2 exactly as np.linalg.norm(centroids - feature, axis=1). */
static double orc_dist(orc_engine *e, const double *c, const double *f) {
    return sqrt(0.0 + pw_sqdiff_block(c, f, e->dim));
}

/* Cluster.seal (clustering.py:71-83): rep = featured member nearest the
 * centroid, first minimum = smallest object id; features dropped. */
static void orc_seal(orc_engine *e, orc_cluster *c) {
    if (c->sealed) return;
    if (c->featured.n) {
        double best = 0;
        int64_t bi = 0;
        for (int64_t j = 0; j < c->featured.n; j++) {
            double dj = orc_dist(e, c->centroid, e->feats + c->featured.v[j] * e->dim);
            if (j == 0 || dj < best) {
                best = dj;
                bi = j;
            }
        }
        c->rep = c->featured_oid.v[bi];
    }
    free(c->sum);
    c->sum = NULL;
    c->sealed = 1;
}

static void merge_classes(orc_cluster *c, const int32_t *topk, int k) {
    /* Cluster.merge_classes (clustering.py:65-69) */
    for (int r = 0; r < k; r++) {
        int64_t cls = topk[r], rank = r + 1, found = 0;
        for (int64_t j = 0; j < c->cls_rank.n; j += 2) {
            if (c->cls_rank.v[j] == cls) {
                if (rank < c->cls_rank.v[j + 1]) c->cls_rank.v[j + 1] = rank;
                found = 1;
                break;
            }
        }
        if (!found) {
            vpush(&c->cls_rank, cls);
            vpush(&c->cls_rank, rank);
        }
    }
}

/* ClusterEngine.insert (clustering.py:104-132).  `row` indexes the feature
 * array; returns the cluster id joined or seeded. */
ORC_API int64_t orc_insert(orc_engine *e, int64_t row, int64_t oid, int64_t fid, const int32_t *topk,
                           int k) {
    const double *f = e->feats + row * e->dim;
    int64_t target = -1;
    double distance = 0.0;
    if (e->nlive) {
        if (e->dbuf_cap < e->nlive) {
            e->dbuf_cap = e->nlive * 2;
            e->dbuf = (double *)realloc(e->dbuf, sizeof(double) * e->dbuf_cap);
        }
        /* distances are independent per live cluster: threads split the row
         * (bit-identical to the serial loop; each distance is one pairwise sum) */
        if (e->nthreads > 1 && e->nlive * (int64_t)e->dim >= 65536) {
#pragma omp parallel for num_threads(e->nthreads) schedule(static)
            for (int64_t j = 0; j < e->nlive; j++)
                e->dbuf[j] = sqrt(0.0 + pw_sqdiff_block(e->cl[e->live[j]].centroid, f, e->dim));
        } else {
            for (int64_t j = 0; j < e->nlive; j++)
                e->dbuf[j] = orc_dist(e, e->cl[e->live[j]].centroid, f);
        }
        e->distance_computations += e->nlive;
        int64_t idx = 0;
        for (int64_t j = 1; j < e->nlive; j++)
            if (e->dbuf[j] < e->dbuf[idx]) idx = j; /* np.argmin: first minimum */
        /* north-star margin accounting (not a reference quantity): the nearest
         * distance within 1e-5 relative of T, or of the runner-up (a tie) */
        {
            const double d1 = e->dbuf[idx];
            double d2 = INFINITY;
            for (int64_t j = 0; j < e->nlive; j++)
                if (j != idx && e->dbuf[j] < d2) d2 = e->dbuf[j];
            if (fabs(d1 - e->t) <= 1e-5 * e->t) e->margin_t++;
            if (d2 - d1 <= 1e-5 * d1) e->margin_tie++;
        }
        if (e->dbuf[idx] <= e->t) {
            target = e->live[idx];
            distance = e->dbuf[idx];
        }
    }
    if (target < 0) {
        if (e->ncl == e->capcl) {
            e->capcl = e->capcl ? e->capcl * 2 : 16;
            e->cl = (orc_cluster *)realloc(e->cl, sizeof(orc_cluster) * e->capcl);
        }
        target = e->ncl++;
        orc_cluster *c = &e->cl[target];
        memset(c, 0, sizeof(*c));
        c->rep = -1;
        c->centroid = (double *)malloc(sizeof(double) * e->dim);
        memcpy(c->centroid, f, sizeof(double) * e->dim);
        if (e->nlive == e->caplive) {
            e->caplive = e->caplive ? e->caplive * 2 : 16;
            e->live = (int64_t *)realloc(e->live, sizeof(int64_t) * e->caplive);
        }
        e->live[e->nlive++] = target;
    }
    orc_cluster *c = &e->cl[target];
    /* Cluster._add (clustering.py:49-59) */
    vpush(&c->members, oid);
    vpush(&c->frames, fid);
    fpush(&c->ins_dist, distance);
    vpush(&c->featured, row);
    vpush(&c->featured_oid, oid);
    if (!c->sum) {
        c->sum = (double *)malloc(sizeof(double) * e->dim);
        memcpy(c->sum, f, sizeof(double) * e->dim);
    } else {
        for (int j = 0; j < e->dim; j++) c->sum[j] += f[j];
    }
    double nf = (double)c->featured.n;
    for (int j = 0; j < e->dim; j++) c->centroid[j] = c->sum[j] / nf;
    if (topk) merge_classes(c, topk, k);
    if (e->nlive > e->m) {
        /* _evict_smallest (clustering.py:139-144): first live of minimum size */
        int64_t vi = 0;
        for (int64_t j = 1; j < e->nlive; j++)
            if (e->cl[e->live[j]].members.n < e->cl[e->live[vi]].members.n) vi = j;
        int64_t victim = e->live[vi];
        memmove(e->live + vi, e->live + vi + 1, sizeof(int64_t) * (e->nlive - vi - 1));
        e->nlive--;
        orc_seal(e, &e->cl[victim]);
    }
    return target;
}

/* ClusterEngine.add_dedup_member (clustering.py:134-137). */
ORC_API void orc_add_dedup(orc_engine *e, int64_t cid, int64_t oid, int64_t fid) {
    orc_cluster *c = &e->cl[cid];
    vpush(&c->members, oid);
    vpush(&c->frames, fid);
}

/* ClusterEngine.finalize (clustering.py:146-153). */
ORC_API void orc_finalize(orc_engine *e) {
    for (int64_t j = 0; j < e->nlive; j++) orc_seal(e, &e->cl[e->live[j]]);
    e->nlive = 0;
}

ORC_API int64_t orc_n_clusters(orc_engine *e) { return e->ncl; }
ORC_API int64_t orc_n_live(orc_engine *e) { return e->nlive; }
ORC_API int64_t orc_distance_computations(orc_engine *e) { return e->distance_computations; }
/* [objects whose nearest distance is within 1e-5 relative of T, ... of a tie] */
ORC_API void orc_margin_counts(orc_engine *e, int64_t out[2]) {
    out[0] = e->margin_t;
    out[1] = e->margin_tie;
}

/* sizes: [n_members, n_featured, rep, n_classes] */
ORC_API void orc_cluster_info(orc_engine *e, int64_t cid, int64_t out[4]) {
    orc_cluster *c = &e->cl[cid];
    out[0] = c->members.n;
    out[1] = c->featured.n;
    out[2] = c->rep;
    out[3] = c->cls_rank.n / 2;
}

ORC_API void orc_cluster_export(orc_engine *e, int64_t cid, double *centroid, int64_t *oids,
                                int64_t *fids, double *ins_dist, int32_t *classes, int32_t *ranks) {
    orc_cluster *c = &e->cl[cid];
    if (centroid) memcpy(centroid, c->centroid, sizeof(double) * e->dim);
    if (oids) memcpy(oids, c->members.v, sizeof(int64_t) * c->members.n);
    if (fids) memcpy(fids, c->frames.v, sizeof(int64_t) * c->frames.n);
    if (ins_dist) memcpy(ins_dist, c->ins_dist.v, sizeof(double) * c->ins_dist.n);
    for (int64_t j = 0; j < c->cls_rank.n / 2; j++) {
        if (classes) classes[j] = (int32_t)c->cls_rank.v[2 * j];
        if (ranks) ranks[j] = (int32_t)c->cls_rank.v[2 * j + 1];
    }
}

/* ingest_stream's object loop (ingest.py:64-76) over a whole stream whose
 * top-K rows (n x k, rows of duplicates ignored) and dup flags are given.
 * out_cluster[i] = cluster the object joined (dups: predecessor's cluster). */
ORC_API orc_engine *orc_ingest(int64_t n, int dim, const int64_t *oids, const int64_t *fids,
                               const double *feats, const int32_t *topk, int k, const uint8_t *is_dup,
                               double t, int64_t m, int64_t *out_cluster) {
    orc_engine *e = orc_engine_new(dim, t, m, feats);
    int64_t prev_cluster = -1;
    for (int64_t i = 0; i < n; i++) {
        if (i > 0 && is_dup[i]) {
            orc_add_dedup(e, prev_cluster, oids[i], fids[i]);
        } else {
            prev_cluster = orc_insert(e, i, oids[i], fids[i], topk ? topk + i * k : NULL, k);
        }
        if (out_cluster) out_cluster[i] = prev_cluster;
    }
    orc_finalize(e);
    return e;
}
