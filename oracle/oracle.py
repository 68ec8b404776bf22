"""CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_1801_03493_b200) never does.

It restates the reference `focusidx` hot path (/root/reference/pkg/src/focusidx):
the float64 / RNG / pairwise-sum arithmetic lives in focus_oracle.c (built to
liboracle.so, see the Makefile); the small integer parts (filler tables, index
build, lookup, query) are numpy restatements here.  Every function cites the
reference line it restates.  Parity of this oracle is pinned by
tests/test_oracle.py against the golden vectors in tests/golden/, which
tools/gen_golden.py produced by running the reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OTHER_CLASS = -1  # core.py:18
GROUND_TRUTH = "GROUND_TRUTH"
GENERIC_CHEAP = "GENERIC_CHEAP"
SPECIALIZED = "SPECIALIZED"

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile liboracle.so (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "focus_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_pairwise_sum.restype = ctypes.c_double
        L.orc_pairwise_sum.argtypes = [_f64p, ctypes.c_int64]
        L.orc_first_uniform3.restype = ctypes.c_double
        L.orc_first_uniform3.argtypes = [ctypes.c_uint64] * 3
        L.orc_first_u64.restype = ctypes.c_uint64
        L.orc_first_u64.argtypes = [_u64p, ctypes.c_int]
        L.orc_rank_from_uniform.restype = ctypes.c_int64
        L.orc_rank_from_uniform.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_int64]
        L.orc_ranks.restype = None
        L.orc_ranks.argtypes = [ctypes.c_int64, ctypes.c_uint64, _i64p, _u8p, ctypes.c_int,
                                ctypes.c_double, ctypes.c_double, ctypes.c_int64, _i32p]
        L.orc_dup_flags.restype = None
        L.orc_dup_flags.argtypes = [ctypes.c_int64, ctypes.c_int, _i64p, _f64p, ctypes.c_double, _u8p]
        L.orc_ingest.restype = ctypes.c_void_p
        L.orc_ingest.argtypes = [ctypes.c_int64, ctypes.c_int, _i64p, _i64p, _f64p, _i32p,
                                 ctypes.c_int, _u8p, ctypes.c_double, ctypes.c_int64, _i64p]
        L.orc_set_threads.restype = None
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_engine_free.restype = None
        L.orc_engine_free.argtypes = [ctypes.c_void_p]
        for name in ("orc_n_clusters", "orc_distance_computations", "orc_n_live"):
            getattr(L, name).restype = ctypes.c_int64
            getattr(L, name).argtypes = [ctypes.c_void_p]
        L.orc_margin_counts.restype = None
        L.orc_margin_counts.argtypes = [ctypes.c_void_p, _i64p]
        L.orc_cluster_info.restype = None
        L.orc_cluster_info.argtypes = [ctypes.c_void_p, ctypes.c_int64, _i64p]
        L.orc_cluster_export.restype = None
        L.orc_cluster_export.argtypes = [ctypes.c_void_p, ctypes.c_int64, _f64p, _i64p, _i64p,
                                         _f64p, _i32p, _i32p]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """Host threads for the per-insert distance row (results are identical)."""
    lib().orc_set_threads(int(n))


def _p(a, t):
    return a.ctypes.data_as(t)


# -- numpy primitives --------------------------------------------------------

def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_pairwise_sum(_p(a, _f64p), a.size)


def first_uniform(seed: int, oid: int, word: int) -> float:
    """First default_rng([seed, oid, word]).random() (classifiers.py:132-133)."""
    return lib().orc_first_uniform3(seed, oid, word)


def first_u64(ints) -> int:
    a = np.asarray(ints, dtype=np.uint64)
    return lib().orc_first_u64(_p(a, _u64p), a.size)


# -- classifier (classifiers.py) ---------------------------------------------

@dataclass(frozen=True)
class Profile:
    """The fields of ClassifierProfile (classifiers.py:73-107) the path reads."""
    profile_id: str
    kind: str
    vocab: int
    p1: float
    rho: float
    cost_units: float
    feature_noise_sigma: float = 0.0
    class_set: tuple | None = None

    @property
    def output_length(self) -> int:  # classifiers.py:92-94
        return len(self.class_set) if self.class_set is not None else self.vocab

    def map_class(self, c: int) -> int:  # classifiers.py:103-107
        if self.class_set is not None and c not in self.class_set:
            return OTHER_CLASS
        return c


def default_profiles(vocab: int = 1000) -> dict:
    """make_default_profiles (classifiers.py:200-204)."""
    gt = Profile("gt", GROUND_TRUTH, vocab, 1.0, 0.0, 58.0)
    cheap = Profile("cheap", GENERIC_CHEAP, vocab, 0.7, 0.95, 58.0 / 8.0, 0.05)
    return {"gt": gt, "cheap": cheap}


def rank_from_uniform(u: float, p1: float, rho: float, out_len: int) -> int:
    return lib().orc_rank_from_uniform(u, p1, rho, out_len)


def ranks(profile: Profile, seed: int, oids, has_label) -> np.ndarray:
    oids = np.ascontiguousarray(oids, dtype=np.int64)
    hl = np.ascontiguousarray(has_label, dtype=np.uint8)
    out = np.empty(oids.size, dtype=np.int32)
    lib().orc_ranks(oids.size, seed, _p(oids, _i64p), _p(hl, _u8p),
                    1 if profile.kind == GROUND_TRUTH else 0, profile.p1, profile.rho,
                    profile.output_length, _p(out, _i32p))
    return out


def confusion_order(kind, vocab, class_set, seed, emitted_true) -> tuple:
    """_confusion_order (classifiers.py:110-123), via numpy's Generator.permutation
    (third-party numpy 2.3.5, the arithmetic the reference itself calls)."""
    rng = np.random.default_rng([seed, 0x0C0F, emitted_true + 1])
    if class_set is None:
        pool = np.arange(vocab)
        pool = pool[pool != emitted_true]
        return tuple(pool[rng.permutation(pool.size)].tolist())
    rest = np.array([c for c in class_set if c != emitted_true and c != OTHER_CLASS])
    tail = tuple(rest[rng.permutation(rest.size)].tolist())
    if emitted_true == OTHER_CLASS:
        return tail
    return (OTHER_CLASS,) + tail


def classify_topk(profile: Profile, seed: int, oids, true_class, k: int) -> np.ndarray:
    """classify(...).top(k).classes() for each object (classifiers.py:136-149,
    core.py:60-61).  true_class < -1 marks an unlabeled object (raises)."""
    oids = np.asarray(oids, dtype=np.int64)
    tc = np.asarray(true_class, dtype=np.int64)
    has = tc >= -1
    if not has.all():
        raise ValueError(f"MissingTrueClass: object {int(oids[~has][0])} has no true class")
    rk = ranks(profile, seed, oids, has)
    out = np.empty((oids.size, k), dtype=np.int32)
    cache = {}
    for i in range(oids.size):
        et = profile.map_class(int(tc[i]))
        if et not in cache:
            cache[et] = confusion_order(profile.kind, profile.vocab, profile.class_set, seed, et)
        fill = cache[et]
        r = int(rk[i])
        classes = fill[: r - 1] + (et,) + fill[r - 1:]
        out[i] = classes[:k]
    return out


def extract_features(profile: Profile, seed: int, oids, feats) -> np.ndarray:
    """extract_feature (classifiers.py:152-158) for every row, float64."""
    sigma = profile.feature_noise_sigma
    feats = np.asarray(feats, dtype=np.float64)
    if sigma == 0.0:
        return feats.copy()
    out = np.empty_like(feats)
    for i, oid in enumerate(np.asarray(oids, dtype=np.int64).tolist()):
        rng = np.random.default_rng([seed, oid, 1])
        out[i] = feats[i] + sigma * rng.standard_normal(feats.shape[1])
    return out


# -- ingest (ingest.py, clustering.py) ---------------------------------------

def dup_flags(fids, sigs, eps: float) -> np.ndarray:
    fids = np.ascontiguousarray(fids, dtype=np.int64)
    sigs = np.ascontiguousarray(sigs, dtype=np.float64)
    n = fids.size
    out = np.zeros(n, dtype=np.uint8)
    s = sigs.shape[1] if sigs.ndim == 2 else 0
    lib().orc_dup_flags(n, s, _p(fids, _i64p), _p(sigs, _f64p), eps, _p(out, _u8p))
    return out.astype(bool)


@dataclass
class OracleCluster:
    cluster_id: int
    centroid: np.ndarray
    member_object_ids: list
    frame_ids: list
    class_best_rank: dict
    centroid_member_id: int | None
    insertion_distances: list = field(default_factory=list)


@dataclass
class OracleIngest:
    is_dup: np.ndarray
    topk: np.ndarray          # n x k (rows of dups are zero)
    cluster_of: np.ndarray    # per object
    clusters: list
    distance_computations: int
    objects_seen: int
    objects_classified: int
    margin_t: int = 0    # nearest distance within 1e-5 relative of T (north-star margin accounting)
    margin_tie: int = 0  # runner-up within 1e-5 relative of the nearest (a tie)


def ingest(oids, fids, sigs, feats, topk, k: int, t: float, m: int, pixel_eps: float = 0.01,
           is_dup=None, with_centroids: bool = True) -> OracleIngest:
    """ingest_stream's clustering part (ingest.py:50-96) on arrays.  `feats`
    are the post-extraction features (float64 or float32), `topk` an n x k
    int32 array of class ids (OTHER = -1) for the classified rows."""
    oids = np.ascontiguousarray(oids, dtype=np.int64)
    fids = np.ascontiguousarray(fids, dtype=np.int64)
    n = oids.size
    if is_dup is None:
        is_dup = dup_flags(fids, sigs, pixel_eps)
    dup = np.ascontiguousarray(is_dup, dtype=np.uint8)
    f64 = np.ascontiguousarray(feats, dtype=np.float64)
    dim = f64.shape[1] if f64.ndim == 2 else 0
    tk = np.ascontiguousarray(topk, dtype=np.int32)
    out = np.empty(n, dtype=np.int64)
    L = lib()
    if n == 0:
        return OracleIngest(dup.astype(bool), tk, out, [], 0, 0, 0)
    h = L.orc_ingest(n, dim, _p(oids, _i64p), _p(fids, _i64p), _p(f64, _f64p), _p(tk, _i32p), k,
                     _p(dup, _u8p), t, m, _p(out, _i64p))
    try:
        clusters = []
        info = np.empty(4, dtype=np.int64)
        for cid in range(L.orc_n_clusters(h)):
            L.orc_cluster_info(h, cid, _p(info, _i64p))
            nm, nf, rep, nc = (int(x) for x in info)
            cen = np.empty(dim, dtype=np.float64)
            mo = np.empty(nm, dtype=np.int64)
            mf = np.empty(nm, dtype=np.int64)
            ins = np.empty(nf, dtype=np.float64)
            cl = np.empty(nc, dtype=np.int32)
            rk = np.empty(nc, dtype=np.int32)
            L.orc_cluster_export(h, cid, _p(cen, _f64p), _p(mo, _i64p), _p(mf, _i64p), _p(ins, _f64p),
                                 _p(cl, _i32p), _p(rk, _i32p))
            clusters.append(OracleCluster(cid, cen if with_centroids else None, mo.tolist(), mf.tolist(),
                                          dict(zip(cl.tolist(), rk.tolist())),
                                          None if rep < 0 else rep, ins.tolist()))
        dc = L.orc_distance_computations(h)
        mg = np.zeros(2, dtype=np.int64)
        L.orc_margin_counts(h, _p(mg, _i64p))
    finally:
        L.orc_engine_free(h)
    classified = int(n - dup[1:].sum()) if n else 0
    return OracleIngest(dup.astype(bool), tk, out, clusters, dc, n, classified, int(mg[0]), int(mg[1]))


# -- index (index.py:60-85) --------------------------------------------------

def build_postings(clusters) -> dict:
    """index.build postings: class -> sorted unique cluster ids."""
    postings: dict = {}
    seen = set()
    for c in clusters:
        if c.cluster_id in seen:
            raise ValueError(f"DuplicateClusterId: {c.cluster_id}")
        seen.add(c.cluster_id)
        for cls in c.class_best_rank:
            postings.setdefault(cls, []).append(c.cluster_id)
    return {cls: sorted(set(v)) for cls, v in postings.items()}


def lookup(clusters_by_id: dict, postings: dict, k: int, class_id: int, k_x=None) -> list:
    if k_x is None:
        k_x = k
    if not 1 <= k_x <= k:
        raise ValueError(f"KxTooLarge: k_x={k_x} outside [1, {k}]")
    ids = postings.get(class_id, [])
    if k_x == k:
        return list(ids)
    return [c for c in ids if clusters_by_id[c].class_best_rank[class_id] <= k_x]


# -- query (query.py:75-137) -------------------------------------------------

class OracleSession:
    """QuerySession restated on arrays; gt_label maps object id -> label."""

    def __init__(self, clusters, k: int, vocab: int, gt_label: dict, gt_cost: float = 58.0,
                 ingest_profile: Profile | None = None):
        self.by_id = {c.cluster_id: c for c in clusters}
        self.postings = build_postings(clusters)
        self.k = k
        self.vocab = vocab
        self.gt = gt_label
        self.gt_cost = gt_cost
        self.ingest_profile = ingest_profile
        self.cache: dict = {}

    def gt_inferences_total(self) -> int:
        return len(self.cache)

    def _verify(self, cid):
        rep = self.by_id[cid].centroid_member_id
        if rep in self.cache:
            return self.cache[rep], False
        label = self.gt[rep]
        if label is None:
            raise ValueError(f"MissingTrueClass: object {rep} has no true class")
        self.cache[rep] = label
        return label, True

    def _matches(self, label, queried):
        if queried == OTHER_CLASS:
            p = self.ingest_profile
            if p is None or p.kind != SPECIALIZED:
                raise ValueError("UnknownClass")
            return p.map_class(label) == OTHER_CLASS
        return label == queried

    def _check(self, c):
        if c != OTHER_CLASS and not 0 <= c < self.vocab:
            raise ValueError(f"UnknownClass: {c}")

    def _collect(self, cids, queried, time_range, keep_label=None):
        frames, objs = [], []
        fresh_n = matched = 0
        for cid in cids:
            label, fresh = self._verify(cid)
            fresh_n += fresh
            ok = (label == keep_label) if keep_label is not None else self._matches(label, queried)
            if not ok:
                continue
            matched += 1
            c = self.by_id[cid]
            mo = np.asarray(c.member_object_ids, dtype=np.int64)
            mf = np.asarray(c.frame_ids, dtype=np.int64)
            if time_range is not None:
                sel = (mf >= time_range[0]) & (mf <= time_range[1])
                mo, mf = mo[sel], mf[sel]
            frames.append(mf)
            objs.append(mo)
        fr = np.unique(np.concatenate(frames)) if frames else np.empty(0, np.int64)
        ob = np.unique(np.concatenate(objs)) if objs else np.empty(0, np.int64)
        return dict(frame_ids=tuple(fr.tolist()), object_ids=tuple(ob.tolist()),
                    gt_inferences=fresh_n, query_cost_units=fresh_n * self.gt_cost,
                    clusters_examined=len(cids), clusters_matched=matched)

    def execute_query(self, class_id, k_x=None, time_range=None):
        self._check(class_id)
        cids = lookup(self.by_id, self.postings, self.k, class_id, k_x)
        return self._collect(cids, class_id, time_range)

    def route_query(self, class_id, k_x=None, time_range=None):
        p = self.ingest_profile
        if (p is not None and p.kind == SPECIALIZED and class_id != OTHER_CLASS
                and class_id not in p.class_set):
            self._check(class_id)
            cids = lookup(self.by_id, self.postings, self.k, OTHER_CLASS, None)
            return self._collect(cids, OTHER_CLASS, time_range, keep_label=class_id)
        return self.execute_query(class_id, k_x, time_range)


# ---------------------------------------------------------------------------
# K1b FC classifier head (north star kernel 1).  There
# is no reference function: the head is a classify_fn for the reference's
# plugin point (ingest.py:52-61,73).  This is its float64 restatement.
# ---------------------------------------------------------------------------

def fc_logits(feats, W, b=None) -> np.ndarray:
    """logits = f W^T + b in float64 (fp32 inputs upcast, as numpy would)."""
    L = np.asarray(feats, np.float64) @ np.asarray(W, np.float64).T
    if b is not None:
        L = L + np.asarray(b, np.float64)
    return L


def fc_topk(feats, W, b, k: int, rel_margin: float = 1e-9):
    """Top-k classes by descending float64 logit, ties -> smaller class id
    (stable sort of -logit).  Also returns a flag per object where two logits
    among ranks 1..k+1 are within rel_margin * max(1, |logit|) of each other --
    the objects whose order depends on float64 rounding (BLAS summation order
    here, the device's own order there), excluded from bit-exact comparison."""
    L = fc_logits(feats, W, b)
    order = np.argsort(-L, axis=1, kind="stable")
    top = order[:, :k].astype(np.int32)
    kk = min(k + 1, L.shape[1])
    vals = np.take_along_axis(L, order[:, :kk], axis=1)
    gaps = vals[:, :-1] - vals[:, 1:]
    scale = np.maximum(1.0, np.abs(vals[:, :-1]))
    flag = (gaps <= rel_margin * scale).any(axis=1) if kk > 1 else np.zeros(L.shape[0], bool)
    return top, flag


def fc_classify_fn(W, b=None):
    """A classify_fn(profile, obj, seed) for the reference ingest_stream that
    ranks classes with the FC head on the object's (already extracted, float32)
    feature: the reference pipeline then runs unchanged on the head's top-K."""
    def fn(profile, obj, seed):
        from focusidx.core import RankedClassification  # reference type, imported lazily
        f = np.asarray(obj.feature, np.float32)
        L = fc_logits(f[None, :], W, b)[0]
        order = np.argsort(-L, kind="stable")
        m = L.max()
        conf = np.exp(L[order] - m) / np.sum(np.exp(L - m))
        return RankedClassification(tuple((int(c), float(p)) for c, p in zip(order, conf)), f)
    return fn
