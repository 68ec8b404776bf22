"""ctypes binding of libfocus_b200.so (include/focus_b200.h).

This is the same binding a maintainer would add to the reference package
(INTEGRATION.md).  There is deliberately no fallback: if the library is not
built or no CUDA device is present, every compute call raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors
from ._build import LIB

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_f64p = ctypes.POINTER(ctypes.c_double)
vp = ctypes.c_void_p

FX_F32, FX_F64 = 0, 1
FX_E_NEED_LABELS = 70
FX_FEATS_COMPACT = 1


class StreamConfig(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("sig_dim", ctypes.c_int32), ("vocab", ctypes.c_int32),
                ("k", ctypes.c_int32), ("t", ctypes.c_double), ("m", ctypes.c_int64),
                ("pixel_eps", ctypes.c_double), ("feat_type", ctypes.c_int32), ("device", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("partition", ctypes.c_int32)]


class RankModelC(ctypes.Structure):
    _fields_ = [("ground_truth", ctypes.c_int32), ("reserved", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("thresholds", c_u64p), ("emit_map", c_i32p), ("fillers", c_i32p)]


class IngestReportC(ctypes.Structure):
    _fields_ = [("objects_seen", ctypes.c_int64), ("objects_classified", ctypes.c_int64),
                ("clusters_emitted", ctypes.c_int64), ("distance_computations", ctypes.c_int64),
                ("gt_invocations", ctypes.c_int64), ("exact_rechecks", ctypes.c_int64)]


class IndexSizes(ctypes.Structure):
    _fields_ = [("n_clusters", ctypes.c_int64), ("dim", ctypes.c_int64), ("n_members", ctypes.c_int64),
                ("n_class_entries", ctypes.c_int64), ("n_postings", ctypes.c_int64), ("vocab", ctypes.c_int64),
                ("k", ctypes.c_int64), ("has_centroids", ctypes.c_int64)]


class QueryResultC(ctypes.Structure):
    _fields_ = [("n_frames", ctypes.c_int64), ("n_objects", ctypes.c_int64), ("gt_inferences", ctypes.c_int64),
                ("clusters_examined", ctypes.c_int64), ("clusters_matched", ctypes.c_int64),
                ("error_cluster", ctypes.c_int64)]


_lib = None

_SIGS = {
    "fx_last_error": (ctypes.c_char_p, []),
    "fx_version": (ctypes.c_int, []),
    "fx_kernel_launches": (ctypes.c_int64, []),
    "fx_stream_create": (ctypes.c_int, [ctypes.POINTER(StreamConfig), ctypes.POINTER(vp)]),
    "fx_stream_destroy": (ctypes.c_int, [vp]),
    "fx_stream_set_rank_model": (ctypes.c_int, [vp, ctypes.POINTER(RankModelC)]),
    "fx_stream_set_fc_head": (ctypes.c_int, [vp, ctypes.c_int32, vp, vp]),
    "fx_fc_topk": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp,
                                  vp, c_i32p, vp, c_u8p]),
    "fx_fc_topk_device": (ctypes.c_int, [ctypes.c_int32, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, vp, vp, vp, vp, vp, vp]),
    "fx_extract_features": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, c_i64p, vp, ctypes.c_int32,
                                           ctypes.c_double, ctypes.c_uint64, c_f64p, c_i64p]),
    "fx_extract_features_device": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, vp, vp,
                                                  ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64,
                                                  vp, ctypes.c_int64, vp, vp]),
    "fx_stream_set_feature_noise": (ctypes.c_int, [vp, ctypes.c_double, ctypes.c_uint64, ctypes.c_int32]),
    "fx_device_set_partitions": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, c_i32p]),
    "fx_dup_flags": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, c_i64p, c_f64p, ctypes.c_double,
                                    c_u8p]),
    "fx_stream_dup_flags": (ctypes.c_int, [vp, ctypes.c_int64, c_i64p, c_f64p, c_u8p]),
    "fx_ingest": (ctypes.c_int, [vp, ctypes.c_int64, c_i64p, c_i64p, c_f64p, vp, c_i32p, c_i32p, ctypes.c_int32]),
    "fx_ingest_rows": (ctypes.c_int, [vp, ctypes.c_int64, c_i64p, c_i64p, c_f64p, vp, ctypes.c_int64, c_i32p, c_i32p]),
    "fx_ingest_device": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp, ctypes.c_int32]),
    "fx_finalize": (ctypes.c_int, [vp, ctypes.POINTER(vp), ctypes.POINTER(IngestReportC)]),
    "fx_stream_object_results": (ctypes.c_int, [vp, c_i32p, c_u8p, c_i32p]),
    "fx_stream_timings": (ctypes.c_int, [vp, c_f64p, ctypes.c_int]),
    "fx_stream_set_timing": (ctypes.c_int, [vp, ctypes.c_int32]),
    "fx_stream_counters": (ctypes.c_int, [vp, c_i64p, ctypes.c_int]),
    "fx_stream_cuda_stream": (ctypes.c_void_p, [vp]),
    "fx_debug_screen_tc": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, vp, vp,
                                          vp]),
    "fx_index_sizes_get": (ctypes.c_int, [vp, ctypes.POINTER(IndexSizes)]),
    "fx_index_export": (ctypes.c_int, [vp, c_i64p, c_f64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i32p, c_i32p,
                                       c_i64p, c_i64p]),
    "fx_index_build": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                      c_i64p, c_f64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i32p, c_i32p,
                                      ctypes.POINTER(vp)]),
    "fx_index_destroy": (ctypes.c_int, [vp]),
    "fx_stream_file_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(vp)]),
    "fx_stream_file_header": (ctypes.c_int, [vp, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)]),
    "fx_stream_file_read": (ctypes.c_int, [vp, c_i64p, c_i64p, c_i32p, c_f64p, vp, ctypes.c_int32, ctypes.c_int32]),
    "fx_stream_file_close": (ctypes.c_int, [vp]),
    "fx_index_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                      ctypes.c_int32, c_i64p, c_f64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i32p,
                                      c_i32p, c_i64p, c_i64p, ctypes.c_int32]),
    "fx_index_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(vp)]),
    "fx_index_file_header": (ctypes.c_int, [vp, ctypes.c_char_p, ctypes.c_int64, c_i64p]),
    "fx_index_file_parse": (ctypes.c_int, [vp, ctypes.c_int64]),
    "fx_index_file_sizes": (ctypes.c_int, [vp, c_i64p]),
    "fx_index_file_export": (ctypes.c_int, [vp, c_i64p, c_i64p, c_i64p, c_f64p, c_i64p, c_i64p, c_i64p, c_i64p,
                                            c_i64p, c_i32p, c_i32p, c_i32p, c_i64p, c_i64p]),
    "fx_index_file_free": (ctypes.c_int, [vp]),
    "fx_lookup": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, c_i64p, ctypes.c_int64, c_i64p]),
    "fx_session_create": (ctypes.c_int, [vp, c_i32p, c_i32p, ctypes.c_int64, c_u8p, ctypes.POINTER(vp)]),
    "fx_session_destroy": (ctypes.c_int, [vp]),
    "fx_query": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(QueryResultC)]),
    "fx_query_fetch": (ctypes.c_int, [vp, c_i64p, c_i64p]),
    "fx_query_fetch_device": (ctypes.c_int, [vp, vp, vp]),
    "fx_session_reset": (ctypes.c_int, [vp]),
    "fx_session_set_labels": (ctypes.c_int, [vp, ctypes.c_int64, c_i32p, c_i32p]),
    "fx_session_gather_labels": (ctypes.c_int, [vp, c_i32p, ctypes.c_int64, ctypes.c_int64]),
    "fx_session_needed": (ctypes.c_int, [vp, c_i32p, c_i64p]),
    "fx_session_seen_open": (ctypes.c_int, [vp, c_i32p]),
    "fx_session_seen_close": (ctypes.c_int, [vp, ctypes.c_int32]),
    "fx_rank_positions": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, c_i64p, c_i32p, ctypes.c_uint64, ctypes.c_int32,
                                         ctypes.c_int32, c_u64p, c_i32p, ctypes.c_int32, ctypes.c_int32, c_i32p,
                                         c_i32p]),
    "fx_index_reps": (ctypes.c_int, [vp, c_i64p]),
    "fx_session_gt_total": (ctypes.c_int64, [vp]),
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB):
    """Load the library (no device access).  Raises DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise errors.DeviceError(f"native library {path} is not built; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status == 0:
        return
    msg = (load().fx_last_error() or b"").decode(errors="replace")
    cls = errors.STATUS.get(status, errors.DeviceError)
    raise cls(msg)


def p64(a: np.ndarray):
    return a.ctypes.data_as(c_i64p)


def p32(a: np.ndarray):
    return a.ctypes.data_as(c_i32p)


def pu8(a: np.ndarray):
    return a.ctypes.data_as(c_u8p)


def pu64(a: np.ndarray):
    return a.ctypes.data_as(c_u64p)


def pf64(a: np.ndarray):
    return a.ctypes.data_as(c_f64p)


def pv(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


_device = int(os.environ.get("FOCUS_B200_DEVICE", "0"))


def set_device(i: int) -> None:
    global _device
    _device = int(i)


def device() -> int:
    return _device
