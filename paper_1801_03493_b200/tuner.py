"""Tuner grid evaluation on the B200.

Drop-in for the reference's cached grid evaluator ``_GridEvaluator``
(focusidx/tuner.py:169-293): same constructor, same ``evaluate(profile, k,
t) -> ConfigEvaluation``, evaluations identical to the reference's (and so,
by test_tuner.py:117-129, to running ingest + query config by config).  What
moved to the device:

  * pixel differencing of the sample (K0, ``fx_dup_flags``);
  * the cluster skeleton of every (noise sigma, T): the ingest engine itself
    (K2 screen / resolve / fold / seal) on the sample's extracted features
    with no class posted -- RankedClassification((), feature) in the
    reference (tuner.py:222-226) -- so one device pass replaces the
    per-object ClusterEngine.insert loop;
  * the class positions of every profile (tuner.py:243-256): the reference
    classifies each object over the full ranked output and searches it; the
    device derives the position from the object's rank (K1a's draw) and the
    emitted class's confusion order (csrc/tuner.cu).
The precision / recall arithmetic (segment sets, macro averages) is the
reference's evaluation harness restated on the host; it is set bookkeeping
over a few thousand frames.

Switch it in the reference with ``focusidx.tuner._GridEvaluator =
paper_1801_03493_b200.tuner.GridEvaluator`` (tests/dropin_plugin.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib, classifiers
from ._reftypes import shared
from .classifiers import GENERIC_CHEAP, GROUND_TRUTH, ClassifierProfile, RankModel, ground_truth_label
from .core import OTHER_CLASS, AccuracyTarget, Config, encode_class
from .errors import EmptySample, UsageError
from .ingest import DEFAULT_PIXEL_EPS, dup_flags, ingest_arrays


@dataclass(frozen=True)
class ConfigEvaluation:  # tuner.py:52-63
    cfg: Config
    est_recall: float
    est_precision: float
    ingest_cost: float
    query_cost: float
    viable: bool

    def cost_sum(self) -> float:
        return self.ingest_cost + self.query_cost


ConfigEvaluation = shared("tuner", "ConfigEvaluation", ConfigEvaluation)


# -- segment-level accuracy (evaluation.py:20-87), host bookkeeping ------------

class SegmentIndex:
    """Object-bearing frames per one-second segment and the GT classes seen in
    them; a class is present in a segment when it is reported in at least
    half (inclusive) of the segment's object-bearing frames."""

    def __init__(self, objects, fps: float):
        self.seg_len = max(1, int(round(fps)))
        self.seg_frames: dict = {}
        self._class_frames: dict = {}
        for o in objects:
            seg = o.frame_id // self.seg_len
            self.seg_frames.setdefault(seg, set()).add(o.frame_id)
            self._class_frames.setdefault(seg, {}).setdefault(ground_truth_label(o), set()).add(o.frame_id)

    def gt_segments(self, class_id: int) -> set:
        return {seg for seg, frames in self.seg_frames.items()
                if (hit := self._class_frames.get(seg, {}).get(class_id)) is not None and 2 * len(hit) >= len(frames)}

    def claimed_segments(self, frame_ids) -> set:
        count: dict = {}
        for fid in set(frame_ids):
            seg = fid // self.seg_len
            if fid in self.seg_frames.get(seg, ()):
                count[seg] = count.get(seg, 0) + 1
        return {seg for seg, c in count.items() if 2 * c >= len(self.seg_frames[seg])}


def class_precision_recall(claimed: set, truth: set) -> tuple:
    hit = len(claimed & truth)
    return (hit / len(claimed) if claimed else 1.0), (hit / len(truth) if truth else 1.0)


def dominant_classes(objects, coverage: float = 0.95) -> list:
    """Fewest GT classes covering `coverage` of the objects (count desc, id asc)."""
    hist: dict = {}
    for o in objects:
        lab = ground_truth_label(o)
        hist[lab] = hist.get(lab, 0) + 1
    out, cum, need = [], 0, coverage * len(objects)
    for cls, cnt in sorted(hist.items(), key=lambda kv: (-kv[1], kv[0])):
        out.append(cls)
        cum += cnt
        if cum >= need:
            break
    return out


def find_gt_profile(profiles) -> ClassifierProfile:
    for p in profiles.values():
        if p.kind == GROUND_TRUTH:
            return p
    raise UsageError("profile registry has no GROUND_TRUTH profile")


# -- device tables for the positions -------------------------------------------

@lru_cache(maxsize=16)
def _position_tables(kind, vocab, class_set, p1, rho, seed):
    """(thresholds u64[out_len-1], emit map i32[V], inverse confusion order
    i32[(V+1) x (V+1)]: index of class c in the fillers of emitted class e,
    -1 if absent), classes encoded (OTHER = V)."""
    V = vocab
    out_len = V if class_set is None else len(class_set)
    if kind == GROUND_TRUTH or out_len <= 1:
        thr = np.zeros(0, np.uint64)
    else:
        thr = np.array(classifiers.rank_thresholds(p1, rho, out_len, out_len - 1), np.uint64)
    members = None if class_set is None else set(class_set)
    emit = np.array([c if members is None or c in members else V for c in range(V)], np.int32)
    inv = np.full((V + 1, V + 1), -1, np.int32)
    emitted = range(V) if class_set is None else [encode_class(c, V) for c in class_set]
    for e in emitted:
        et = OTHER_CLASS if e == V else e
        fill = classifiers._filler_prefix(kind, vocab, class_set, seed, et, out_len)
        inv[e, [encode_class(c, V) for c in fill]] = np.arange(len(fill), dtype=np.int32)
    return thr, emit, inv


class _Skeleton:
    """Cluster structure of one (sigma, T) (tuner.py:154-166)."""

    def __init__(self, row_cluster, rep_label, frames):
        self.row_cluster = row_cluster
        self.rep_label = rep_label
        self.frames = frames
        self.n_clusters = len(frames)
        self._by_class: dict = {}

    def clusters_of_class(self, cls: int) -> np.ndarray:
        if cls not in self._by_class:
            self._by_class[cls] = np.flatnonzero(self.rep_label == cls)
        return self._by_class[cls]


class GridEvaluator:
    """Drop-in for focusidx.tuner._GridEvaluator (tuner.py:169-293)."""

    def __init__(self, header, sample, profiles, targets: AccuracyTarget, pixel_eps: float = DEFAULT_PIXEL_EPS,
                 seed: int = 0, m: int = 100):
        self.header = header
        self.sample = list(sample)
        if not self.sample:
            raise EmptySample("empty tuning sample")
        self.targets = targets
        self.pixel_eps = pixel_eps
        self.seed = seed
        self.m = m
        self._gt_prof = find_gt_profile(profiles)
        self.gt_cost = self._gt_prof.cost_units
        self.segidx = SegmentIndex(self.sample, header.fps)
        self.dominant = dominant_classes(self.sample)
        self._gt_segs = {c: self.segidx.gt_segments(c) for c in self.dominant}
        n = len(self.sample)
        self._oids = np.fromiter((o.object_id for o in self.sample), np.int64, n)
        self._fids = np.fromiter((o.frame_id for o in self.sample), np.int64, n)
        S = len(self.sample[0].pixel_signature)
        self._sigs = np.array([o.pixel_signature for o in self.sample], np.float64).reshape(n, S)
        self.is_dup = dup_flags(self._fids, self._sigs, pixel_eps)  # K0 (ingest.py:37-47)
        self._keep = np.flatnonzero(~self.is_dup)
        self.classified = [self.sample[i] for i in self._keep.tolist()]
        self.n_classified = len(self.classified)
        self._labels = {o.object_id: o for o in self.sample}
        self._features: dict = {}
        self._skeletons: dict = {}
        self._pos: dict = {}

    def _features_for(self, sigma: float) -> np.ndarray:
        if sigma not in self._features:
            stub = ClassifierProfile("_noise", GENERIC_CHEAP, self.header.vocab, RankModel(0.5, 0.5), 1.0,
                                     feature_noise_sigma=sigma)
            # extract_feature (classifiers.py:152-158) for the whole sample on the device
            D = self.header.dim
            raw = [np.asarray(o.feature) for o in self.classified]
            dt = np.float32 if raw and all(r.dtype == np.float32 for r in raw) else np.float64
            R = np.array(raw, dtype=dt).reshape(self.n_classified, D) if raw else np.zeros((0, D), dt)
            oids = np.array([o.object_id for o in self.classified], np.int64)
            F = classifiers.extract_features(stub, oids, R, self.seed) if raw else np.zeros((0, D))
            self._features[sigma] = F.reshape(self.n_classified, D)
        return self._features[sigma]

    def _skeleton_for(self, sigma: float, t: float) -> _Skeleton:
        key = (sigma, t)
        if key in self._skeletons:
            return self._skeletons[key]
        F = self._features_for(sigma)
        if np.array_equal(F.astype(np.float32).astype(np.float64), F):
            F = F.astype(np.float32)
        n = len(self.sample)
        cfg = Config("_skeleton", k=1, l_s=self.header.vocab, t=t, m=self.m)
        # features only: every top-K slot empty (-1), no class is posted
        topk = np.full((n, 1), -1, np.int32)
        idx, _, st = ingest_arrays(self._oids, self._fids, self._sigs, F, cfg, self._gt_prof, vocab=self.header.vocab,
                                   pixel_eps=self.pixel_eps, topk=topk, compact=True)
        cl, _, _ = st.object_results(n, 1)
        ex = idx.device.export(centroids=False)
        row_cluster = cl[self._keep].astype(np.int64)  # cluster ids are 0..C-1 = finalize order
        rep_label = np.array([ground_truth_label(self._labels[int(r)]) for r in ex["reps"].tolist()], np.int64)
        mo, mf = ex["mem_off"], ex["mem_fid"]
        frames = [set(mf[mo[i]:mo[i + 1]].tolist()) for i in range(ex["cluster_ids"].size)]
        skel = _Skeleton(row_cluster, rep_label, frames)
        self._skeletons[key] = skel
        return skel

    def _positions(self, profile: ClassifierProfile, class_id: int) -> np.ndarray:
        key = (profile.profile_id, class_id)
        if key not in self._pos:
            # every dominant class's lookup class of this profile in one launch
            want = sorted({c if (profile.class_set is None or c in profile.class_set) else OTHER_CLASS
                           for c in self.dominant} | {class_id})
            thr, emit, inv = _position_tables(profile.kind, profile.vocab, profile.class_set,
                                              profile.rank_model.p1, profile.rank_model.rho, self.seed)
            V = profile.vocab
            emitted = np.array([emit[ground_truth_label(o)] if 0 <= ground_truth_label(o) < V else V
                                for o in self.classified], np.int32)
            cls = np.array([encode_class(c, V) for c in want], np.int32)
            out = np.empty((cls.size, self.n_classified), np.int32)
            inv_c = np.ascontiguousarray(inv)
            oids = np.ascontiguousarray(self._oids[self._keep])
            _lib.check(_lib.load().fx_rank_positions(
                _lib.device(), self.n_classified, _lib.p64(oids), _lib.p32(emitted),
                ctypes.c_uint64(self.seed & ((1 << 64) - 1)), 1 if profile.kind == GROUND_TRUTH else 0, thr.size,
                thr.ctypes.data_as(_lib.c_u64p), _lib.p32(inv_c), V + 1, cls.size, _lib.p32(cls), _lib.p32(out)))
            for q, c in enumerate(want):
                self._pos[(profile.profile_id, c)] = out[q].astype(np.int64)
        return self._pos[key]

    def evaluate(self, profile: ClassifierProfile, k: int, t: float) -> ConfigEvaluation:
        """tuner.py:258-293: per dominant class, the clusters hit by the class
        at rank < k, kept when their representative's GT label is the class;
        segment precision / recall of their frames; macro averages."""
        skel = self._skeleton_for(profile.feature_noise_sigma, t)
        precisions, recalls, costs = [], [], []
        for cls in self.dominant:
            direct = profile.class_set is None or cls in profile.class_set
            pos = self._positions(profile, cls if direct else OTHER_CLASS)
            matched = np.bincount(skel.row_cluster[pos < k], minlength=skel.n_clusters) > 0
            verified = skel.clusters_of_class(cls)
            verified = verified[matched[verified]]
            frames: set = set()
            for ci in verified:
                frames.update(skel.frames[ci])
            p, r = class_precision_recall(self.segidx.claimed_segments(frames), self._gt_segs[cls])
            precisions.append(p)
            recalls.append(r)
            costs.append(int(np.count_nonzero(matched)) * self.gt_cost)
        n = len(self.dominant)
        est_precision = sum(precisions) / n
        est_recall = sum(recalls) / n
        cfg = Config(profile_id=profile.profile_id, k=k, l_s=profile.l_s, t=t, m=self.m, targets=self.targets)
        return ConfigEvaluation(cfg=cfg, est_recall=est_recall, est_precision=est_precision,
                                ingest_cost=self.n_classified * profile.cost_units, query_cost=sum(costs) / n,
                                viable=(est_recall >= self.targets.recall_target
                                        and est_precision >= self.targets.precision_target))


__all__ = ["GridEvaluator", "ConfigEvaluation", "SegmentIndex", "class_precision_recall", "dominant_classes"]
