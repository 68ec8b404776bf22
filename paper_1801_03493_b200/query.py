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
from .classifiers import GROUND_TRUTH, SPECIALIZED
from .core import OTHER_CLASS, encode_class
from .errors import MissingTrueClass, NonMonotoneSchedule, UnknownClass


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


_NO_LABEL, _NO_OBJECT, _NO_REP = -2, -3, -4


class QuerySession:
    """Read-only device index + the verification oracle for one session."""

    def __init__(self, idx, gt_profile, objects, ingest_profile=None, labels=None):
        if gt_profile.kind != GROUND_TRUTH:
            raise UnknownClass(f"{gt_profile.profile_id!r} is not a GT profile")
        self.idx = idx
        self.gt_profile = gt_profile
        self.objects = objects
        self.ingest_profile = ingest_profile
        self.L = _lib.load()
        ex = idx.device.export(centroids=False)
        reps = ex["reps"]
        C = reps.size
        label = np.empty(C, np.int32)
        key = np.empty(C, np.int32)
        keys = {}
        for i, r in enumerate(reps.tolist()):
            if r < 0:
                label[i] = _NO_REP
                key[i] = keys.setdefault(("none", i), len(keys))
                continue
            key[i] = keys.setdefault(r, len(keys))
            if labels is not None:
                label[i] = labels[r]
                continue
            obj = objects.get(r) if hasattr(objects, "get") else None
            if obj is None and r not in objects:
                label[i] = _NO_OBJECT
            else:
                obj = objects[r]
                label[i] = _NO_LABEL if obj.true_class is None else obj.true_class
        self._rep_label = label
        other = None
        V = idx.header.vocab
        if ingest_profile is not None and ingest_profile.kind == SPECIALIZED:
            cs = set(ingest_profile.class_set)
            other = np.array([0 if c in cs else 1 for c in range(V)], np.uint8)
        h = _lib.vp()
        _lib.check(self.L.fx_session_create(idx.device.handle, _lib.p32(label), _lib.p32(key), len(keys),
                                            _lib.pu8(other) if other is not None else None, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h is not None and _lib._lib is not None:
            _lib._lib.fx_session_destroy(h)

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
        kx = -1 if k_x is None else int(k_x)
        st = self.L.fx_query(self.handle, enc, kx, mode, int(keep_label), batch_step, 1 if has else 0, t0, t1,
                             ctypes.byref(res))
        if st == 20:  # MissingTrueClass names the representative object
            rep = self.idx.device.export(centroids=False)["reps"][res.error_cluster]
            raise MissingTrueClass(f"object {int(rep)} has no true class")
        if st == 60:
            rep = self.idx.device.export(centroids=False)["reps"][res.error_cluster]
            raise KeyError(int(rep))
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
        for i, kx in enumerate(sched):
            yield self._run(req.class_id, kx, 0, 0, 1 if i == 0 else 2, req.time_range)
