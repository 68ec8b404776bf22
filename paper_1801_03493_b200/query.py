"""Query: the drop-in QuerySession (focusidx/query.py:19-154) on the B200.

lookup with k_x, GT verification of one representative per candidate
cluster (a label gather, memoised per session by representative object id)
and member expansion into sorted unique frame / object ids all run in
csrc/query.cu.  Routing (OTHER, query_other, batched schedules) and the
exceptions are the reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._reftypes import shared
from .classifiers import GROUND_TRUTH, SPECIALIZED
from .core import OTHER_CLASS, encode_class
from .errors import KxTooLarge, MissingTrueClass, NonMonotoneSchedule, UnknownClass


@dataclass(frozen=True)
class QueryRequest:
    class_id: int
    k_x: int | None = None
    time_range: tuple | None = None


@dataclass(frozen=True)
class QueryResult:
    frame_ids: tuple
    object_ids: tuple
    gt_inferences: int
    query_cost_units: float
    clusters_examined: int
    clusters_matched: int


QueryRequest = shared("query", "QueryRequest", QueryRequest)
QueryResult = shared("query", "QueryResult", QueryResult)

_NO_LABEL, _NO_OBJECT, _NO_REP = -2, -3, -4


class QuerySession:
    """Read-only device index + the verification oracle for one session.

    Construction is O(1) in Python: GT labels of representatives are produced
    lazily, like the reference's ``_verify`` (query.py:53-60) -- the device
    query lists the candidates whose label it does not know yet, the session
    reads just those from ``objects`` and re-issues the query (nothing is
    applied before that).  ``labels`` (optional, not a reference argument): a
    dense array of GT labels indexed by object id (-2 = unlabeled), gathered
    for every representative on the device in one pass.
    """

    def __init__(self, idx, gt_profile, objects, ingest_profile=None, labels=None):
        if gt_profile.kind != GROUND_TRUTH:
            raise UnknownClass(f"{gt_profile.profile_id!r} is not a GT profile")
        self.idx = idx
        self.gt_profile = gt_profile
        self.objects = objects
        self.ingest_profile = ingest_profile
        self._labels = labels
        self.L = _lib.load()
        dev = idx.ensure_device()  # e.g. index.load(): posted on the device once
        C = int(dev.sizes.n_clusters)
        reps = getattr(dev, "_reps_cache", None)  # built indexes are immutable: read once
        if reps is None:
            reps = np.empty(C, np.int64)
            if C:
                _lib.check(self.L.fx_index_reps(dev.handle, _lib.p64(reps)))
            dev._reps_cache = reps
        self._reps = reps
        # memo key = representative object id (query.py:53-60); representatives
        # of distinct clusters are distinct objects unless the index was built
        # by hand, in which case equal representatives share one key
        key, n_keys = None, C
        have = reps[reps >= 0]
        if np.unique(have).size != have.size:
            _, inv = np.unique(np.where(reps >= 0, reps, -1 - np.arange(C)), return_inverse=True)
            key, n_keys = inv.astype(np.int32), int(inv.max()) + 1 if C else 0
        other = None
        V = idx.header.vocab
        if ingest_profile is not None and ingest_profile.kind == SPECIALIZED:
            other = np.ones(V, np.uint8)
            cs = np.array([c for c in ingest_profile.class_set if 0 <= c < V], np.int64)
            other[cs] = 0
        rl = None
        if isinstance(labels, np.ndarray) and C:
            # the representatives' labels only (C values, not the whole array),
            # handed to the session when it is created
            lab = np.asarray(labels)
            ok = (reps >= 0) & (reps < lab.size)
            rl = np.full(C, _NO_OBJECT, np.int32)
            rl[ok] = lab[reps[ok]]
            rl[reps < 0] = _NO_REP
        h = _lib.vp()
        _lib.check(self.L.fx_session_create(dev.handle, None if rl is None else _lib.p32(rl),
                                            None if key is None else _lib.p32(key), n_keys,
                                            _lib.pu8(other) if other is not None else None, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h is not None and _lib._lib is not None:
            _lib._lib.fx_session_destroy(h)

    def _label_of(self, r: int) -> int:
        """ground_truth_label(objects[r]) encoded (classifiers.py:161-165)."""
        if r < 0:
            return _NO_REP
        src = self._labels if self._labels is not None else self.objects
        if self._labels is not None:
            lab = src.get(r, _NO_OBJECT) if hasattr(src, "get") else _NO_OBJECT
            return _NO_LABEL if lab is None else int(lab)
        try:
            obj = src[r]
        except (KeyError, IndexError, TypeError):
            return _NO_OBJECT
        return _NO_LABEL if obj.true_class is None else int(obj.true_class)

    def _supply_labels(self) -> None:
        n = ctypes.c_int64(0)
        _lib.check(self.L.fx_session_needed(self.handle, None, ctypes.byref(n)))
        cidx = np.empty(n.value, np.int32)
        _lib.check(self.L.fx_session_needed(self.handle, _lib.p32(cidx), ctypes.byref(n)))
        lab = np.fromiter((self._label_of(r) for r in self._reps[cidx].tolist()), np.int32, cidx.size)
        _lib.check(self.L.fx_session_set_labels(self.handle, cidx.size, _lib.p32(cidx), _lib.p32(lab)))

    def gt_inferences_total(self) -> int:
        return int(self.L.fx_session_gt_total(self.handle))

    def _check_class(self, class_id: int) -> None:
        if class_id != OTHER_CLASS and not 0 <= class_id < self.idx.header.vocab:
            raise UnknownClass(str(class_id))

    def reset(self) -> None:
        """Forget every verification: the session is as fresh as a new one."""
        _lib.check(self.L.fx_session_reset(self.handle))

    def _launch(self, class_id, k_x, mode, keep_label, batch_step, time_range):
        V = self.idx.header.vocab
        enc = encode_class(class_id, V)
        res = _lib.QueryResultC()
        has = time_range is not None
        t0, t1 = (int(time_range[0]), int(time_range[1])) if has else (0, 0)
        K = self.idx.header.k
        kx = K if (k_x is None or mode == 1) else k_x
        if not 1 <= kx <= K:  # index.lookup (index.py:77-80)
            raise KxTooLarge(f"k_x={kx} outside [1, {K}]")
        while True:
            st = self.L.fx_query(self.handle, enc, int(kx), mode, int(keep_label), batch_step, 1 if has else 0,
                                 t0, t1, ctypes.byref(res))
            if st != _lib.FX_E_NEED_LABELS:
                break
            self._supply_labels()
        if st == 20:  # MissingTrueClass names the representative object
            rep = int(self._reps[res.error_cluster])
            raise MissingTrueClass(f"object {rep} has no true class")
        if st == 60:
            rep = int(self._reps[res.error_cluster])
            raise KeyError(None if rep < 0 else rep)
        _lib.check(st)
        return res

    def query_device(self, req: QueryRequest, out_frames=None, out_objects=None):
        """execute_query with the frame / object ids left in device memory:
        returns (n_frames, n_objects, stats); when torch device tensors (int64,
        large enough) are given the ids are copied into them.  stats =
        (gt_inferences, clusters_examined, clusters_matched)."""
        self._check_class(req.class_id)
        res = self._launch(req.class_id, req.k_x, 0, 0, 0, req.time_range)
        if out_frames is not None or out_objects is not None:
            _lib.check(self.L.fx_query_fetch_device(
                self.handle, None if out_frames is None else _lib.vp(out_frames.data_ptr()),
                None if out_objects is None else _lib.vp(out_objects.data_ptr())))
        return int(res.n_frames), int(res.n_objects), (int(res.gt_inferences), int(res.clusters_examined),
                                                       int(res.clusters_matched))

    def fetch_device(self, out_frames, out_objects) -> None:
        """Copy the last query's ids into torch int64 device tensors."""
        _lib.check(self.L.fx_query_fetch_device(self.handle, _lib.vp(out_frames.data_ptr()),
                                                _lib.vp(out_objects.data_ptr())))

    def query_arrays(self, req: QueryRequest):
        """execute_query returning numpy int64 arrays (frames, objects) + stats."""
        self._check_class(req.class_id)
        res = self._launch(req.class_id, req.k_x, 0, 0, 0, req.time_range)
        fr = np.empty(res.n_frames, np.int64)
        ob = np.empty(res.n_objects, np.int64)
        if res.n_frames or res.n_objects:
            _lib.check(self.L.fx_query_fetch(self.handle, _lib.p64(fr), _lib.p64(ob)))
        return fr, ob, (int(res.gt_inferences), int(res.clusters_examined), int(res.clusters_matched))

    def _run(self, class_id, k_x, mode, keep_label, batch_step, time_range) -> QueryResult:
        res = self._launch(class_id, k_x, mode, keep_label, batch_step, time_range)
        fr = np.empty(res.n_frames, np.int64)
        ob = np.empty(res.n_objects, np.int64)
        if res.n_frames or res.n_objects:
            _lib.check(self.L.fx_query_fetch(self.handle, _lib.p64(fr), _lib.p64(ob)))
        return QueryResult(frame_ids=tuple(fr.tolist()), object_ids=tuple(ob.tolist()),
                           gt_inferences=int(res.gt_inferences),
                           query_cost_units=int(res.gt_inferences) * self.gt_profile.cost_units,
                           clusters_examined=int(res.clusters_examined), clusters_matched=int(res.clusters_matched))

    def execute_query(self, req: QueryRequest) -> QueryResult:
        self._check_class(req.class_id)
        return self._run(req.class_id, req.k_x, 0, 0, 0, req.time_range)

    def query_other(self, raw_class: int, time_range=None) -> QueryResult:
        self._check_class(raw_class)
        p = self.ingest_profile
        if p is None or p.kind != SPECIALIZED:
            raise UnknownClass("query_other requires a specialized ingest profile")
        if raw_class in p.class_set:
            return self.execute_query(QueryRequest(raw_class, time_range=time_range))
        return self._run(OTHER_CLASS, None, 1, raw_class, 0, time_range)

    def route_query(self, class_id: int, k_x=None, time_range=None) -> QueryResult:
        p = self.ingest_profile
        if (p is not None and p.kind == SPECIALIZED and class_id != OTHER_CLASS
                and class_id not in p.class_set):
            return self.query_other(class_id, time_range=time_range)
        return self.execute_query(QueryRequest(class_id, k_x=k_x, time_range=time_range))

    def batched_query(self, req: QueryRequest, batch_schedule):
        sched = list(batch_schedule)
        if not sched or any(b <= a for a, b in zip(sched, sched[1:])):
            raise NonMonotoneSchedule(str(sched))
        self._check_class(req.class_id)
        sid = ctypes.c_int32(0)
        _lib.check(self.L.fx_session_seen_open(self.handle, ctypes.byref(sid)))
        try:  # this generator's own seen set (query.py:149)
            for kx in sched:
                yield self._run(req.class_id, kx, 0, 0, sid.value + 1, req.time_range)
        finally:
            if getattr(self, "handle", None) is not None:
                self.L.fx_session_seen_close(self.handle, sid.value)
