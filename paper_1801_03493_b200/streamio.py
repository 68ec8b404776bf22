"""FOCUSSTREAM/1 stream files (drop-in for focusidx.streamio; SURVEY.md §8f
row 3).  Decoding -- 2,048 text floats per object line dominate file-based
ingest -- runs in the native library with host threads
(fx_stream_file_*); `read_stream_arrays` hands flat arrays straight to
`ingest_arrays`, `read_stream` rebuilds the reference's DetectedObject list.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .core import DetectedObject, encode_class
from .ingest import StreamHeader

_MAGIC = "FOCUSSTREAM/1"


def _csv(vec) -> str:
    return ",".join(f"{x:.9g}" for x in vec)


def write_stream(path, header: StreamHeader, objects) -> None:
    """streamio.write_stream (streamio.py:43-55)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"{_MAGIC}\n")
        fh.write(f"stream_id={header.stream_id}\n")
        fh.write(f"fps={header.fps:.9g}\n")
        fh.write(f"D={header.dim}\n")
        fh.write(f"S={header.sig_dim}\n")
        fh.write(f"V={header.vocab}\n")
        fh.write("[OBJECTS]\n")
        for obj in objects:
            cls = "" if obj.true_class is None else str(encode_class(obj.true_class, header.vocab))
            fh.write(f"{obj.object_id}|{obj.frame_id}|{cls}|{_csv(obj.pixel_signature)}|{_csv(obj.feature)}\n")


def read_stream_arrays(path, feat_dtype=np.float64, threads: int = 0):
    """Decode a stream file into (StreamHeader, dict of arrays): object_ids,
    frame_ids (int64), true_class (int32; OTHER = -1, unlabeled = -2),
    pixel_signatures (n x S float64), features (n x D, float64 or float32).
    Raises what read_stream raises (FormatVersionMismatch, DataError,
    ValueError) for the first bad line."""
    L = _lib.load()
    h = _lib.vp()
    _lib.check(L.fx_stream_file_open(os.fsencode(path), ctypes.byref(h)))
    try:
        sid = ctypes.create_string_buffer(4096)
        fps = ctypes.c_double()
        D, S, V = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        n = ctypes.c_int64()
        _lib.check(L.fx_stream_file_header(h, sid, len(sid), ctypes.byref(fps), ctypes.byref(D), ctypes.byref(S),
                                           ctypes.byref(V), ctypes.byref(n)))
        header = StreamHeader(stream_id=sid.value.decode("utf-8"), fps=fps.value, dim=D.value, sig_dim=S.value,
                              vocab=V.value)
        f32 = np.dtype(feat_dtype) == np.float32
        out = dict(object_ids=np.empty(n.value, np.int64), frame_ids=np.empty(n.value, np.int64),
                   true_class=np.empty(n.value, np.int32),
                   pixel_signatures=np.empty((n.value, max(S.value, 0)), np.float64),
                   features=np.empty((n.value, max(D.value, 0)), np.float32 if f32 else np.float64))
        _lib.check(L.fx_stream_file_read(h, _lib.p64(out["object_ids"]), _lib.p64(out["frame_ids"]),
                                         _lib.p32(out["true_class"]), _lib.pf64(out["pixel_signatures"]),
                                         out["features"].ctypes.data_as(ctypes.c_void_p), 1 if f32 else 0,
                                         int(threads)))
    finally:
        L.fx_stream_file_close(h)
    return header, out


def read_stream(path):
    """streamio.read_stream (streamio.py:58-113): (StreamHeader, [DetectedObject])."""
    header, a = read_stream_arrays(path)
    objects = []
    for i in range(len(a["object_ids"])):
        tc = int(a["true_class"][i])
        fid = int(a["frame_ids"][i])
        objects.append(DetectedObject(object_id=int(a["object_ids"][i]), frame_id=fid,
                                      timestamp_s=fid / header.fps, pixel_signature=a["pixel_signatures"][i],
                                      feature=a["features"][i], true_class=None if tc == -2 else tc))
    return header, objects


__all__ = ["write_stream", "read_stream", "read_stream_arrays"]
