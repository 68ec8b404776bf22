"""Classifier profiles and the device tables of the cheap-CNN rank model.

Profiles, the rank model and specialization mirror the reference
(classifiers.py:43-107, 168-204).  The per-object classification itself --
the SeedSequence/PCG64 draw, the rank and the top-K splice
(classifiers.py:126-149) -- runs on the device (K1a, csrc/ingest.cu); this
module only derives the per-profile tables it needs:

  * rank thresholds: for j = 0..K-1 the smallest 53-bit integer u with
    rank_from_uniform(u * 2^-53) >= j + 2.  The rank is monotone in u, so a
    binary search with the reference formula (same libm `log`) yields tables
    that reproduce its ranks bit-exactly on the device;
  * the first K fillers of every emitted class's confusion order
    (numpy Generator.permutation, as classifiers.py:110-123 draws it);
  * the emit map (true class -> emitted class, OTHER for out-of-set classes).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from ._reftypes import shared
from .core import OTHER_CLASS, DetectedObject, encode_class
from .errors import DataError, DimensionMismatch, EmptyHistogram, MissingTrueClass, UsageError

GROUND_TRUTH = "GROUND_TRUTH"
GENERIC_CHEAP = "GENERIC_CHEAP"
SPECIALIZED = "SPECIALIZED"

GT_COST = 58.0
GENERIC_COST = GT_COST / 8.0
SPECIALIZE_COST_FACTOR = 10.0
SPECIALIZE_RHO_FACTOR = 0.8

_U53 = 1 << 53
NO_THRESHOLD = (1 << 64) - 1


@dataclass(frozen=True)
class RankModel:
    """Inclusion curve p(k) = 1 - (1 - p1) * rho**(k - 1)."""
    p1: float
    rho: float

    def __post_init__(self):
        if not (0 < self.p1 <= 1):
            raise DataError(f"p1={self.p1} outside (0, 1]")
        if not (0 <= self.rho < 1):
            raise DataError(f"rho={self.rho} outside [0, 1)")

    def inclusion(self, k: int) -> float:
        return 1.0 - (1.0 - self.p1) * self.rho ** (k - 1)

    def rank_from_uniform(self, u: float, output_length: int) -> int:
        """Smallest k with p(k) >= u, capped at the output length."""
        if output_length == 1 or u <= self.p1:
            return 1
        if self.rho == 0.0:
            return min(2, output_length)
        steps = math.floor(math.log((1.0 - u) / (1.0 - self.p1)) / math.log(self.rho))
        return min(max(2 + steps, 2), output_length)


@dataclass(frozen=True)
class ClassifierProfile:
    profile_id: str
    kind: str
    vocab: int
    rank_model: RankModel
    cost_units: float
    feature_noise_sigma: float = 0.0
    class_set: tuple | None = None

    def __post_init__(self):
        if self.kind == SPECIALIZED:
            if self.class_set is None or OTHER_CLASS not in self.class_set:
                raise DataError("specialized profile needs a class_set containing OTHER")
        elif self.class_set is not None:
            raise DataError("class_set is only valid for SPECIALIZED profiles")
        if self.cost_units <= 0:
            raise DataError("cost_units must be positive")

    @property
    def output_length(self) -> int:
        return self.vocab if self.class_set is None else len(self.class_set)

    @property
    def l_s(self) -> int:
        return self.vocab if self.class_set is None else len(self.class_set) - 1

    def map_class(self, class_id: int) -> int:
        if self.class_set is None or class_id in self.class_set:
            return class_id
        return OTHER_CLASS


RankModel = shared("classifiers", "RankModel", RankModel)
ClassifierProfile = shared("classifiers", "ClassifierProfile", ClassifierProfile)


def make_default_profiles(vocab: int = 1000) -> dict:
    """The 'gt' oracle and the generic 'cheap' model (classifiers.py:200-204)."""
    gt = ClassifierProfile("gt", GROUND_TRUTH, vocab, RankModel(1.0, 0.0), GT_COST)
    cheap = ClassifierProfile("cheap", GENERIC_CHEAP, vocab, RankModel(0.7, 0.95), GENERIC_COST,
                              feature_noise_sigma=0.05)
    return {gt.profile_id: gt, cheap.profile_id: cheap}


def specialize_profile(base: ClassifierProfile, class_histogram: dict, l_s: int,
                       cost_factor: float = SPECIALIZE_COST_FACTOR,
                       rho_factor: float = SPECIALIZE_RHO_FACTOR) -> ClassifierProfile:
    """Keep the l_s most frequent classes (ties -> smaller id) plus OTHER
    (classifiers.py:168-192)."""
    if not class_histogram:
        raise EmptyHistogram("cannot specialize on an empty class histogram")
    if l_s < 1:
        raise DataError(f"l_s={l_s} must be >= 1")
    keep = sorted(sorted(class_histogram, key=lambda c: (-class_histogram[c], c))[:l_s])
    return ClassifierProfile(
        profile_id=f"{base.profile_id}+spec{l_s}", kind=SPECIALIZED, vocab=base.vocab,
        rank_model=RankModel(base.rank_model.p1, base.rank_model.rho * rho_factor),
        cost_units=base.cost_units / cost_factor, feature_noise_sigma=base.feature_noise_sigma,
        class_set=tuple(keep) + (OTHER_CLASS,))


def ground_truth_label(obj: DetectedObject) -> int:
    """The GT-CNN's top-1: the object's stored label (classifiers.py:161-165)."""
    if obj.true_class is None:
        raise MissingTrueClass(f"object {obj.object_id} has no true class")
    return obj.true_class


def extract_feature(profile: ClassifierProfile, obj: DetectedObject, rng_seed: int) -> np.ndarray:
    """The cheap CNN's feature vector (classifiers.py:152-158).  This is the
    ingest INPUT: a real deployment gets it from the
    CNN; the synthetic profile perturbs the stored feature with numpy's
    standard_normal stream of default_rng([seed, object_id, 1])."""
    if profile.feature_noise_sigma == 0.0:
        return np.array(obj.feature, copy=True)
    g = np.random.default_rng([rng_seed, obj.object_id, 1])
    return obj.feature + profile.feature_noise_sigma * g.standard_normal(obj.feature.shape[0])


def extract_features(profile: ClassifierProfile, object_ids, feats, rng_seed: int,
                     device: int | None = None) -> np.ndarray:
    """extract_feature (classifiers.py:152-158) for a batch of objects on the
    device (csrc/noise.cu): row i = feats[i] + sigma * default_rng([rng_seed,
    object_ids[i], 1]).standard_normal(D), float64, bit for bit."""
    from . import _lib
    oids = np.ascontiguousarray(object_ids, np.int64)
    F = np.asarray(feats)
    if F.dtype != np.float32:
        F = F.astype(np.float64, copy=False)
    F = np.ascontiguousarray(F).reshape(oids.size, -1)
    out = np.empty(F.shape, np.float64)
    if profile.feature_noise_sigma == 0.0:
        out[...] = F
        return out
    nflag = np.zeros(1, np.int64)
    _lib.check(_lib.load().fx_extract_features(
        _lib.device() if device is None else device, oids.size, F.shape[1], _lib.p64(oids), _lib.pv(F),
        _lib.FX_F32 if F.dtype == np.float32 else _lib.FX_F64, float(profile.feature_noise_sigma),
        rng_seed & ((1 << 64) - 1), _lib.pf64(out), _lib.p64(nflag)))
    return out


# -- device tables -----------------------------------------------------------

def _rank_of_u53(model: RankModel, out_len: int, u53: int) -> int:
    return model.rank_from_uniform(u53 * (1.0 / 9007199254740992.0), out_len)


@lru_cache(maxsize=256)
def rank_thresholds(p1: float, rho: float, out_len: int, k: int) -> tuple:
    """thr[j] = min u53 with rank >= j + 2 (NO_THRESHOLD if unreachable)."""
    model = RankModel(p1, rho)
    out = []
    for j in range(k):
        want = j + 2
        if _rank_of_u53(model, out_len, _U53 - 1) < want:
            out.append(NO_THRESHOLD)
            continue
        lo, hi = 0, _U53 - 1  # rank(hi) >= want
        while lo < hi:
            mid = (lo + hi) // 2
            if _rank_of_u53(model, out_len, mid) >= want:
                hi = mid
            else:
                lo = mid + 1
        # monotonicity witness at the boundary
        assert _rank_of_u53(model, out_len, lo) >= want
        assert lo == 0 or _rank_of_u53(model, out_len, lo - 1) < want
        out.append(lo)
    return tuple(out)


@lru_cache(maxsize=4096)
def _filler_prefix(kind: str, vocab: int, class_set, seed: int, emitted_true: int, k: int) -> tuple:
    """First k entries of the confusion order (classifiers.py:110-123)."""
    g = np.random.default_rng([seed, 0x0C0F, emitted_true + 1])
    if class_set is None:
        pool = np.arange(vocab)
        pool = pool[pool != emitted_true]
        order = pool[g.permutation(pool.size)]
        return tuple(order[:k].tolist())
    rest = np.array([c for c in class_set if c != emitted_true and c != OTHER_CLASS])
    tail = rest[g.permutation(rest.size)].tolist()
    full = tail if emitted_true == OTHER_CLASS else [OTHER_CLASS] + tail
    return tuple(full[:k])


@lru_cache(maxsize=64)
def _device_tables(kind, vocab, class_set, p1, rho, seed, k):
    V = vocab
    out_len = V if class_set is None else len(class_set)
    if kind == GROUND_TRUTH:
        thr = np.full(k, NO_THRESHOLD, dtype=np.uint64)
    else:
        thr = np.array(rank_thresholds(p1, rho, out_len, k), dtype=np.uint64)
    members = None if class_set is None else set(class_set)
    emit = np.array([c if members is None or c in members else V for c in range(V)], dtype=np.int32)
    fill = np.full((V + 1, k), -1, dtype=np.int32)
    emitted = range(V) if class_set is None else [encode_class(c, V) for c in class_set]
    for e in emitted:
        et = OTHER_CLASS if e == V else e
        pref = _filler_prefix(kind, vocab, class_set, seed, et, k)
        fill[e, :len(pref)] = [encode_class(c, V) for c in pref]
    return thr, emit, fill.reshape(-1)


def device_tables(profile: ClassifierProfile, seed: int, k: int):
    """(thresholds u64[k], emit_map i32[V], fillers i32[(V+1)*k]) for K1a."""
    return _device_tables(profile.kind, profile.vocab, profile.class_set, profile.rank_model.p1,
                          profile.rank_model.rho, seed, k)


class FCHead:
    """K1b: the cheap-CNN classifier head of the north star (no reference
    function; a classify_fn for ingest.py:52-61,73).  logits = f W^T + b over
    W.shape[0] classes; the top-k by descending logit (ties -> smaller class id)
    are the object's ranked classes and the extracted feature is what gets
    clustered.  Runs only on the device: pass it as `classify_fn` to
    ingest_stream, or call `topk` on a batch of feature rows."""

    def __init__(self, W, b=None):
        self.W = np.ascontiguousarray(W, np.float32)
        self.b = None if b is None else np.ascontiguousarray(b, np.float32)
        if self.W.ndim != 2 or (self.b is not None and self.b.shape != (self.W.shape[0],)):
            raise ValueError("W must be (vocab, dim) and b (vocab,)")

    @property
    def vocab(self) -> int:
        return int(self.W.shape[0])

    def topk(self, feats, k: int, device: int | None = None):
        """(topk int32[n, k], confidences float32[n, k], margin flags bool[n]) on the device."""
        from . import _lib
        F = np.ascontiguousarray(feats, np.float32)
        n, D = F.shape
        if D != self.W.shape[1]:
            raise DimensionMismatch(f"feature dim {D} != head dim {self.W.shape[1]}")
        tk = np.empty((n, k), np.int32)
        conf = np.empty((n, k), np.float32)
        flag = np.empty(n, np.uint8)
        L = _lib.load()
        _lib.check(L.fx_fc_topk(_lib.device() if device is None else device, n, D, self.vocab, k, _lib.pv(F),
                                _lib.pv(self.W), None if self.b is None else _lib.pv(self.b), _lib.p32(tk),
                                _lib.pv(conf), _lib.pu8(flag)))
        return tk, conf, flag.astype(bool)

    def __call__(self, profile, obj, seed):
        raise UsageError("FCHead runs on the device: pass it as classify_fn to ingest_stream or call .topk()")
