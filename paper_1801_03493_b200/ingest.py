"""Ingest: the drop-in `ingest_stream` (focusidx/ingest.py:50-96) on the B200.

Control flow is the reference's; the work is not:
  K0 pixel differencing, K1a rank-model top-K, K2 batched screen + exact
  sequential resolve + fold, deferred seal, K3 index build all run in
  libfocus_b200.so.  The host marshals the stream into arrays and raises the
  reference's exceptions.

`classify_fn` (the reference's plugin point, ingest.py:52-61,73) is honoured:
when given, it is called once per retained object in stream order and its
top-K classes and feature are what the device clusters.  When omitted, the
device rank model classifies; the profile's feature noise (extract_feature,
classifiers.py:152-158) is the ingest input -- the cheap CNN's output.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, classifiers
from ._reftypes import shared
from .core import Config, encode_class, validate_config
from .errors import DimensionMismatch, SignatureLengthMismatch
from .index import DeviceIndex, IndexHeader, TopKIndex

DEFAULT_PIXEL_EPS = 0.01


@dataclass(frozen=True)
class IngestReport:
    objects_seen: int
    objects_classified: int
    clusters_emitted: int
    ingest_cost_units: float
    dedup_savings_units: float
    distance_computations: int
    gt_invocations: int = 0


@dataclass(frozen=True)
class StreamHeader:
    """Fields of streamio.StreamHeader (streamio.py:30-36) the path reads."""
    stream_id: str
    fps: float
    dim: int
    sig_dim: int
    vocab: int


IngestReport = shared("ingest", "IngestReport", IngestReport)
StreamHeader = shared("streamio", "StreamHeader", StreamHeader)


class Stream:
    """One device stream engine (one per video stream, single writer)."""

    def __init__(self, dim: int, sig_dim: int, vocab: int, k: int, t: float, m: int,
                 pixel_eps: float = DEFAULT_PIXEL_EPS, feat_type: int = _lib.FX_F32,
                 device: int | None = None, batch: int = 0, partition: int = 0):
        self.L = _lib.load()
        cfg = _lib.StreamConfig(dim=dim, sig_dim=sig_dim, vocab=vocab, k=k, t=float(t), m=int(m),
                                pixel_eps=float(pixel_eps), feat_type=feat_type,
                                device=_lib.device() if device is None else device, batch=batch,
                                partition=partition)
        self.cfg = cfg
        h = _lib.vp()
        _lib.check(self.L.fx_stream_create(ctypes.byref(cfg), ctypes.byref(h)))
        self.handle = h
        self._keep = []

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h is not None and _lib._lib is not None:
            _lib._lib.fx_stream_destroy(h)

    def set_rank_model(self, profile, seed: int):
        thr, emit, fill = classifiers.device_tables(profile, seed, self.cfg.k)
        rm = _lib.RankModelC(ground_truth=1 if profile.kind == classifiers.GROUND_TRUTH else 0,
                             seed=seed & ((1 << 64) - 1), thresholds=_lib.pu64(thr), emit_map=_lib.p32(emit),
                             fillers=_lib.p32(fill))
        _lib.check(self.L.fx_stream_set_rank_model(self.handle, ctypes.byref(rm)))

    def set_fc_head(self, head):
        """Use the K1b FC classifier head (classifiers.FCHead) for top-K."""
        W = np.ascontiguousarray(head.W, np.float32)
        b = None if head.b is None else np.ascontiguousarray(head.b, np.float32)
        self._keep += [W, b]
        _lib.check(self.L.fx_stream_set_fc_head(self.handle, W.shape[0], _lib.pv(W), None if b is None else _lib.pv(b)))

    def set_feature_noise(self, sigma: float, seed: int, in_dtype):
        """The engine clusters extract_feature (classifiers.py:152-158) of the
        raw feature rows fx_ingest receives, computed on the device."""
        it = _lib.FX_F32 if np.dtype(in_dtype) == np.float32 else _lib.FX_F64
        _lib.check(self.L.fx_stream_set_feature_noise(self.handle, float(sigma), seed & ((1 << 64) - 1), it))
        self._noise = sigma != 0.0

    def dup_flags(self, fids: np.ndarray, sigs: np.ndarray) -> np.ndarray:
        n = fids.size
        out = np.zeros(n, np.uint8)
        if n:
            _lib.check(self.L.fx_stream_dup_flags(self.handle, n, _lib.p64(fids), _lib.pf64(sigs), _lib.pu8(out)))
        return out.astype(bool)

    def ingest(self, oids, fids, sigs, feats, true_class=None, topk=None, compact=False):
        n = oids.size
        if compact and not getattr(self, "_noise", False):
            # the row count is known: the feature upload starts before K0 (fx_ingest_rows)
            _lib.check(self.L.fx_ingest_rows(self.handle, n, _lib.p64(oids), _lib.p64(fids), _lib.pf64(sigs),
                                             _lib.pv(feats), int(feats.shape[0]) if feats.ndim == 2 else 0,
                                             _lib.p32(true_class) if true_class is not None else None,
                                             _lib.p32(topk) if topk is not None else None))
            return
        _lib.check(self.L.fx_ingest(self.handle, n, _lib.p64(oids), _lib.p64(fids), _lib.pf64(sigs), _lib.pv(feats),
                                    _lib.p32(true_class) if true_class is not None else None,
                                    _lib.p32(topk) if topk is not None else None,
                                    _lib.FX_FEATS_COMPACT if compact else 0))

    def ingest_device(self, n, oids_ptr, fids_ptr, sigs_ptr, feats_ptr, tcls_ptr=None, topk_ptr=None, compact=False):
        _lib.check(self.L.fx_ingest_device(self.handle, n, oids_ptr, fids_ptr, sigs_ptr, feats_ptr, tcls_ptr,
                                           topk_ptr, _lib.FX_FEATS_COMPACT if compact else 0))

    def finalize(self):
        rep = _lib.IngestReportC()
        h = _lib.vp()
        _lib.check(self.L.fx_finalize(self.handle, ctypes.byref(h), ctypes.byref(rep)))
        return DeviceIndex(h), rep

    def object_results(self, n: int, k: int):
        cl = np.empty(n, np.int32)
        dup = np.empty(n, np.uint8)
        tk = np.empty(n * k, np.int32)
        _lib.check(self.L.fx_stream_object_results(self.handle, _lib.p32(cl), _lib.pu8(dup), _lib.p32(tk)))
        return cl, dup.astype(bool), tk.reshape(n, k)

    COUNTERS = ("nlive", "next_cid", "dc", "nfree", "nevict_total", "exact", "nsnap", "nres", "ninserted",
                "nevict_batch", "ndefer", "nod", "last_cid", "ndirty", "err", "fast", "fc_flagged", "ev_cursor",
                "fast_state", "fast_done", "fast_batches", "noise_flagged", "cyc_passA", "cyc_passB", "cyc_passCD", "cyc_confirm", "cyc_passE", "cyc_seq", "windows", "seq_steps",
                "conf_b0", "conf_b1_7", "conf_b8_15", "conf_b16_31", "conf_b32_63", "conf_b64_127", "conf_b128",
                "conf_young", "fold_wait_cyc", "fold_chain_cyc", "fold_slot_cyc", "fold_rows", "fold_slots")
    PHASES = ("k0_k1a", "screen", "resolve", "fold", "seal", "index", "batches", "screen_resid",
              "host_screen", "host_resolve", "host_ring", "host_fold", "host_grow", "host_k0", "host_k1",
              "screen_summary")

    def set_timing(self, on: bool = True) -> None:
        """Record per-phase CUDA-event timers (off by default: they add gaps)."""
        _lib.check(self.L.fx_stream_set_timing(self.handle, 1 if on else 0))

    def counters(self) -> dict:
        out = np.zeros(len(self.COUNTERS), np.int64)
        _lib.check(self.L.fx_stream_counters(self.handle, _lib.p64(out), out.size))
        return dict(zip(self.COUNTERS, out.tolist()))

    def timings(self) -> dict:
        out = np.zeros(len(self.PHASES), np.float64)
        _lib.check(self.L.fx_stream_timings(self.handle, _lib.pf64(out), out.size))
        return dict(zip(self.PHASES, out.tolist()))

    def cuda_stream(self) -> int:
        return int(self.L.fx_stream_cuda_stream(self.handle) or 0)


def pixel_diff(prev, cur, eps: float) -> bool:
    """ingest.py:37-47 for one pair, evaluated by the device K0 kernel."""
    if eps < 0:
        return False
    a, b = np.asarray(prev.pixel_signature, np.float64), np.asarray(cur.pixel_signature, np.float64)
    if a.shape[0] != b.shape[0]:
        raise SignatureLengthMismatch(f"{a.shape[0]} vs {b.shape[0]}")
    if cur.frame_id - prev.frame_id > 1:
        return False
    return bool(dup_flags(np.array([prev.frame_id, cur.frame_id], np.int64), np.stack([a, b]), eps)[1])


def dup_flags(fids: np.ndarray, sigs: np.ndarray, eps: float, device: int | None = None) -> np.ndarray:
    """K0 over a whole sequence: is_dup[i] = pixel_diff(obj[i-1], obj[i], eps)."""
    fids = np.ascontiguousarray(fids, np.int64)
    n = fids.size
    S = sigs.shape[1] if sigs.ndim == 2 else 0
    sigs = np.ascontiguousarray(sigs, np.float64).reshape(n, S)
    out = np.zeros(n, np.uint8)
    if n:
        _lib.check(_lib.load().fx_dup_flags(_lib.device() if device is None else device, n, S, _lib.p64(fids),
                                            _lib.pf64(sigs), float(eps), _lib.pu8(out)))
    return out.astype(bool)


def _f32_exact(x: np.ndarray) -> bool:
    return x.dtype == np.float32 or bool(np.array_equal(x.astype(np.float32).astype(x.dtype), x))


def ingest_arrays(oids, fids, sigs, feats, cfg: Config, profile, *, vocab: int, seed: int = 0,
                  pixel_eps: float = DEFAULT_PIXEL_EPS, true_class=None, topk=None, compact: bool = False,
                  stream_id: str = "synthetic", device: int | None = None, batch: int = 0, fc_head=None,
                  raw_features: bool = False):
    """Array-level ingest: the C-ABI call with host buffers.  `feats` rows are
    the extracted features (float32 or float64) -- or, with `raw_features`,
    the objects' raw features (compact rows), extracted on the device with the
    profile's noise (classifiers.py:152-158); `true_class` (int32, -2 =
    unlabeled) drives the device rank model, or `topk` (n x k encoded, OTHER =
    V) comes from an external classifier.  Returns (TopKIndex, IngestReport,
    Stream)."""
    oids = np.ascontiguousarray(oids, np.int64)
    fids = np.ascontiguousarray(fids, np.int64)
    n = oids.size
    S = sigs.shape[1] if sigs.ndim == 2 else 0
    sigs = np.ascontiguousarray(sigs, np.float64).reshape(n, S)
    D = feats.shape[1] if feats.ndim == 2 else 0
    feat_type = _lib.FX_F64 if feats.dtype == np.float64 else _lib.FX_F32
    noise = raw_features and profile.feature_noise_sigma != 0.0
    if noise:
        if not compact:
            raise ValueError("raw_features needs compact feature rows")
        feat_type = _lib.FX_F64  # feature + float64 noise is float64 (numpy promotion)
    feats = np.ascontiguousarray(feats)
    st = Stream(D, S, vocab, cfg.k, cfg.t, cfg.m, pixel_eps, feat_type, device, batch)
    if noise:
        st.set_feature_noise(profile.feature_noise_sigma, seed, feats.dtype)
    if fc_head is not None:
        st.set_fc_head(fc_head)
    elif topk is None:
        st.set_rank_model(profile, seed)
    if n:
        st.ingest(oids, fids, sigs, feats,
                  true_class=None if true_class is None else np.ascontiguousarray(true_class, np.int32),
                  topk=None if topk is None else np.ascontiguousarray(topk, np.int32), compact=compact)
    dix, rep = st.finalize()
    header = IndexHeader(stream_id=stream_id, dim=D, vocab=vocab, n_objects=n, config=cfg)
    report = IngestReport(
        objects_seen=rep.objects_seen, objects_classified=rep.objects_classified,
        clusters_emitted=rep.clusters_emitted,
        ingest_cost_units=rep.objects_classified * profile.cost_units,
        dedup_savings_units=(rep.objects_seen - rep.objects_classified) * profile.cost_units,
        distance_computations=rep.distance_computations)
    assert report.distance_computations <= cfg.m * report.objects_classified, "O(Mn) distance budget exceeded"
    return TopKIndex(header, device=dix), report, st


def ingest_stream(header, stream, cfg: Config, profiles, pixel_eps: float = DEFAULT_PIXEL_EPS,
                  seed: int = 0, classify_fn=None):
    """Drop-in for focusidx.ingest.ingest_stream; returns (TopKIndex, IngestReport)."""
    validate_config(cfg, profiles)
    profile = profiles[cfg.profile_id]
    objs = list(stream)
    n = len(objs)
    D, V, K = header.dim, header.vocab, cfg.k
    oids = np.fromiter((o.object_id for o in objs), np.int64, n)
    fids = np.fromiter((o.frame_id for o in objs), np.int64, n)
    slen = [np.shape(o.pixel_signature)[0] for o in objs]
    S = slen[0] if n else 0
    if pixel_eps >= 0:
        for i in range(1, n):
            if slen[i] != slen[i - 1]:
                raise SignatureLengthMismatch(f"{slen[i - 1]} vs {slen[i]}")
    if any(s != S for s in slen):
        # differencing off: signatures are never compared; pad to a common width
        S = max(slen)
    sigs = np.zeros((n, S), np.float64)
    for i, o in enumerate(objs):
        sigs[i, :slen[i]] = o.pixel_signature
    dup = dup_flags(fids, sigs, pixel_eps)
    keep = np.flatnonzero(~dup)
    fc_head = classify_fn if isinstance(classify_fn, classifiers.FCHead) else None
    raw = False
    if fc_head is not None:
        # K1b on the device: the head sees the extracted features and emits top-K
        topk, tcls = None, None
        rows = None
        F = classifiers.extract_features(profile, oids[keep], _raw_rows(objs, keep, D), seed)
    elif classify_fn is not None:
        # -1 = no class at that rank: a classifier may emit fewer than K
        # classes and the reference merges only those (clustering.py:65-69)
        topk = np.full((n, K), -1, np.int32)
        rows = []
        for i in keep.tolist():
            rc = classify_fn(profile, objs[i], seed).top(K)
            cls = [encode_class(c, V) for c in rc.classes()]
            topk[i, :len(cls)] = cls
            rows.append(np.asarray(rc.feature))
        tcls = None
    else:
        # the device rank model classifies; extract_feature runs on the device
        # over the raw rows (the engine's feature-noise stage)
        topk = None
        tcls = np.array([-2 if o.true_class is None else o.true_class for o in objs], np.int32)
        rows = None
        F = _raw_rows(objs, keep, D)
        raw = profile.feature_noise_sigma != 0.0
    if rows is not None:  # classify_fn's features
        for r in rows:
            if np.shape(r)[0] != D:
                raise DimensionMismatch(f"feature dim {np.shape(r)[0]} != engine dim {D}")
        all32 = all(np.asarray(r).dtype == np.float32 for r in rows)
        F = np.array(rows, dtype=np.float64).reshape(len(rows), D) if rows else np.zeros((0, D))
        if all32:
            F = F.astype(np.float32)
    if fc_head is not None:
        F = F.astype(np.float32)  # the K1b head consumes float32 rows
    elif not raw and F.dtype != np.float32 and _f32_exact(F):
        F = F.astype(np.float32)  # float64 values that are float32-exact: the TC screen path
    idx, report, _ = ingest_arrays(oids, fids, sigs, F, cfg, profile, vocab=V, seed=seed, pixel_eps=pixel_eps,
                                   true_class=tcls, topk=topk, compact=True, stream_id=header.stream_id,
                                   fc_head=fc_head, raw_features=raw)
    idx.header = IndexHeader(stream_id=header.stream_id, dim=D, vocab=V, n_objects=n, config=cfg)
    return idx, report


def _raw_rows(objs, keep, D) -> np.ndarray:
    """The retained objects' raw feature rows (float32 if every row is
    float32, else float64 -- numpy's promotion of the stacked rows)."""
    rows = [objs[i].feature for i in keep.tolist()]
    for r in rows:
        if np.shape(r)[0] != D:
            raise DimensionMismatch(f"feature dim {np.shape(r)[0]} != engine dim {D}")
    if not rows:
        return np.zeros((0, D), np.float32)
    dt = np.float32 if all(np.asarray(r).dtype == np.float32 for r in rows) else np.float64
    return np.ascontiguousarray(np.array(rows, dtype=dt).reshape(len(rows), D))
