"""TopKIndex on the device (drop-in for focusidx.index build/lookup).

`build` (index.py:60-72) posts clusters under every class of their class set;
`lookup` (index.py:75-85) filters a class's postings by best rank <= k_x.
Both run on the device (K3 / K4, csrc/index.cu, csrc/capi.cu); the Python
TopKIndex keeps the reference's fields (`header`, `clusters`, `postings`),
materialising them lazily from the device index on first access.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._reftypes import shared
from .clustering import Cluster
import os

from .core import Config, decode_class, encode_class, format_config, parse_config
from .errors import ChecksumMismatch, DataError, DuplicateClusterId, FormatVersionMismatch, KxTooLarge


@dataclass(frozen=True)
class IndexHeader:
    stream_id: str
    dim: int
    vocab: int
    n_objects: int
    config: Config

    @property
    def k(self) -> int:
        return self.config.k


IndexHeader = shared("index", "IndexHeader", IndexHeader)


class DeviceIndex:
    """Owner of an fx_index handle."""

    def __init__(self, handle):
        self.handle = handle
        sz = _lib.IndexSizes()
        _lib.check(_lib.load().fx_index_sizes_get(handle, ctypes.byref(sz)))
        self.sizes = sz
        self._export = None

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h is not None and _lib._lib is not None:
            _lib._lib.fx_index_destroy(h)

    def export(self, centroids: bool = True) -> dict:
        if self._export is not None and (not centroids or "centroids" in self._export):
            return self._export
        s = self.sizes
        C, D = s.n_clusters, s.dim
        out = dict(
            cluster_ids=np.empty(C, np.int64), reps=np.empty(C, np.int64),
            mem_off=np.empty(C + 1, np.int64), mem_oid=np.empty(s.n_members, np.int64),
            mem_fid=np.empty(s.n_members, np.int64), cls_off=np.empty(C + 1, np.int64),
            cls_id=np.empty(s.n_class_entries, np.int32), cls_rank=np.empty(s.n_class_entries, np.int32),
            post_off=np.empty(s.vocab + 2, np.int64), post_cluster=np.empty(s.n_postings, np.int64))
        cen = None
        if centroids and s.has_centroids:
            cen = np.empty((C, D), np.float64)
            out["centroids"] = cen
        _lib.check(_lib.load().fx_index_export(
            self.handle, _lib.p64(out["cluster_ids"]), _lib.pf64(cen) if cen is not None else None,
            _lib.p64(out["reps"]), _lib.p64(out["mem_off"]), _lib.p64(out["mem_oid"]), _lib.p64(out["mem_fid"]),
            _lib.p64(out["cls_off"]), _lib.p32(out["cls_id"]), _lib.p32(out["cls_rank"]),
            _lib.p64(out["post_off"]), _lib.p64(out["post_cluster"])))
        self._export = out
        return out


class TopKIndex:
    """header + clusters (id -> Cluster) + postings (class -> sorted ids)."""

    def __init__(self, header: IndexHeader, clusters=None, postings=None, device: DeviceIndex | None = None,
                 file_arrays: dict | None = None):
        self.header = header
        self._clusters = clusters
        self._postings = postings
        self.device = device
        self._file = file_arrays  # CSR arrays of a loaded FOCUSIDX/1 file (fx_index_file_export)

    def ensure_device(self) -> DeviceIndex:
        """The device index, posted on first use (a loaded or hand-built index)."""
        if self.device is None:
            if self._file is not None and self._clusters is None:
                self.device = _device_from_file(self._file, self.header)
            else:
                self.device = build(list(self.clusters.values()), self.header).device
        return self.device

    # -- lazily materialised reference fields --------------------------------
    @property
    def clusters(self) -> dict:
        if self._clusters is None:
            self._materialise()
        return self._clusters

    @clusters.setter
    def clusters(self, v):
        self._clusters = v

    @property
    def postings(self) -> dict:
        if self._postings is None:
            self._materialise()
        return self._postings

    @postings.setter
    def postings(self, v):
        self._postings = v

    def _materialise(self):
        if self._file is not None:
            return self._materialise_file()
        ex = self.device.export(centroids=True)
        V = self.header.vocab
        cen = ex.get("centroids")
        clusters = {}
        mo, co, ci = ex["mem_off"], ex["cls_off"], ex["cls_id"]
        for i, cid in enumerate(ex["cluster_ids"].tolist()):
            a, b = mo[i], mo[i + 1]
            ca, cb = co[i], co[i + 1]
            ranks = {(-1 if c == V else c): r for c, r in zip(ci[ca:cb].tolist(), ex["cls_rank"][ca:cb].tolist())}
            rep = int(ex["reps"][i])
            clusters[cid] = Cluster(
                cluster_id=cid, centroid=cen[i] if cen is not None else np.zeros(self.header.dim),
                member_object_ids=ex["mem_oid"][a:b].tolist(),
                frame_ids=ex["mem_fid"][a:b].tolist(), class_best_rank=ranks,
                centroid_member_id=None if rep < 0 else rep, sealed=True)
        postings = {}
        po, pc = ex["post_off"], ex["post_cluster"]
        for enc in range(V + 1):
            a, b = po[enc], po[enc + 1]
            if b > a:
                postings[-1 if enc == V else enc] = pc[a:b].tolist()
        if self._clusters is None:
            self._clusters = clusters
        if self._postings is None:
            self._postings = postings

    def _materialise_file(self):
        f = self._file
        clusters = {}
        co, mo, fo, ko = f["cen_off"], f["mem_off"], f["fr_off"], f["cls_off"]
        for i, cid in enumerate(f["cid"].tolist()):
            cm = int(f["cmid"][i])
            clusters[cid] = Cluster(
                cluster_id=cid, centroid=f["cen"][co[i]:co[i + 1]].copy(),
                member_object_ids=f["mem"][mo[i]:mo[i + 1]].tolist(), frame_ids=f["fr"][fo[i]:fo[i + 1]].tolist(),
                class_best_rank=dict(zip(f["cls"][ko[i]:ko[i + 1]].tolist(), f["rank"][ko[i]:ko[i + 1]].tolist())),
                centroid_member_id=None if cm == _NO_CMID else cm, sealed=True)
        po = f["post_off"]
        postings = {c: f["post_ids"][po[j]:po[j + 1]].tolist() for j, c in enumerate(f["post_cls"].tolist())}
        if self._clusters is None:
            self._clusters = clusters
        if self._postings is None:
            self._postings = postings

    def record_count(self) -> int:
        return len(self.clusters) + sum(len(v) for v in self.postings.values())


def build(clusters, header: IndexHeader, device: int | None = None) -> TopKIndex:
    """index.build on the device: clusters are marshalled into CSR arrays
    (sorted by id), postings are built by K3 (csrc/index.cu)."""
    cl = sorted(clusters, key=lambda c: c.cluster_id)
    V, D = header.vocab, header.dim
    C = len(cl)
    ids = np.array([c.cluster_id for c in cl], dtype=np.int64)
    reps = np.array([-1 if c.centroid_member_id is None else c.centroid_member_id for c in cl], dtype=np.int64)
    mem_off = np.zeros(C + 1, np.int64)
    cls_off = np.zeros(C + 1, np.int64)
    for i, c in enumerate(cl):
        mem_off[i + 1] = mem_off[i] + len(c.member_object_ids)
        cls_off[i + 1] = cls_off[i] + len(c.class_best_rank)
    mem_oid = np.fromiter((o for c in cl for o in c.member_object_ids), np.int64, int(mem_off[-1]))
    mem_fid = np.fromiter((f for c in cl for f in c.frame_ids), np.int64, int(mem_off[-1]))
    cls_id = np.fromiter((encode_class(k, V) for c in cl for k in c.class_best_rank), np.int32, int(cls_off[-1]))
    cls_rank = np.fromiter((r for c in cl for r in c.class_best_rank.values()), np.int32, int(cls_off[-1]))
    cen = None
    if C and all(getattr(c, "centroid", None) is not None and np.shape(c.centroid) == (D,) for c in cl):
        cen = np.ascontiguousarray(np.array([c.centroid for c in cl], dtype=np.float64).reshape(C, D))
    L = _lib.load()
    h = _lib.vp()
    _lib.check(L.fx_index_build(C, V, header.k, D, _lib.device() if device is None else device, _lib.p64(ids),
                                _lib.pf64(cen) if cen is not None else None, _lib.p64(reps), _lib.p64(mem_off),
                                _lib.p64(mem_oid), _lib.p64(mem_fid), _lib.p64(cls_off), _lib.p32(cls_id),
                                _lib.p32(cls_rank), ctypes.byref(h)))
    dev = DeviceIndex(h)
    by_id = {c.cluster_id: c for c in cl}
    return TopKIndex(header, clusters=by_id, postings=None, device=dev)


def lookup(idx: TopKIndex, class_id: int, k_x: int | None = None) -> list:
    """Cluster ids posted under class_id with best rank <= k_x, ascending."""
    k = idx.header.k
    kx = k if k_x is None else k_x
    if not 1 <= kx <= k:
        raise KxTooLarge(f"k_x={kx} outside [1, {k}]")
    V = idx.header.vocab
    enc = encode_class(class_id, V)
    if enc < 0 or enc > V:
        return []
    idx.ensure_device()  # e.g. loaded from a file: posted on the device once
    L = _lib.load()
    n = ctypes.c_int64(0)
    _lib.check(L.fx_lookup(idx.device.handle, enc, kx, None, 0, ctypes.byref(n)))
    out = np.empty(n.value, np.int64)
    if n.value:
        _lib.check(L.fx_lookup(idx.device.handle, enc, kx, _lib.p64(out), n.value, ctypes.byref(n)))
    return out.tolist()


# -- serialization: FOCUSIDX/1 (index.py:88-204) ------------------------------

_MAGIC = "FOCUSIDX/1"


def _cluster_arrays(clusters, V: int, D: int) -> dict:
    """fx_index_export layout of Python Cluster records."""
    cl = list(clusters)
    C = len(cl)
    mem_off = np.zeros(C + 1, np.int64)
    cls_off = np.zeros(C + 1, np.int64)
    for i, c in enumerate(cl):
        mem_off[i + 1] = mem_off[i] + len(c.member_object_ids)
        cls_off[i + 1] = cls_off[i] + len(c.class_best_rank)
    return dict(
        cluster_ids=np.array([c.cluster_id for c in cl], np.int64),
        reps=np.array([-1 if c.centroid_member_id is None else c.centroid_member_id for c in cl], np.int64),
        centroids=np.ascontiguousarray(np.array([np.asarray(c.centroid, np.float64) for c in cl],
                                                np.float64).reshape(C, D)),
        mem_off=mem_off,
        mem_oid=np.fromiter((o for c in cl for o in c.member_object_ids), np.int64, int(mem_off[-1])),
        mem_fid=np.fromiter((f for c in cl for f in c.frame_ids), np.int64, int(mem_off[-1])),
        cls_off=cls_off,
        cls_id=np.fromiter((encode_class(k, V) for c in cl for k in c.class_best_rank), np.int32, int(cls_off[-1])),
        cls_rank=np.fromiter((r for c in cl for r in c.class_best_rank.values()), np.int32, int(cls_off[-1])))


def _posting_arrays(postings: dict, V: int) -> dict:
    off = np.zeros(V + 2, np.int64)
    by_enc = {encode_class(c, V): ids for c, ids in postings.items()}
    for enc in range(V + 1):
        off[enc + 1] = off[enc] + len(by_enc.get(enc, ()))
    ids = np.fromiter((x for enc in range(V + 1) for x in by_enc.get(enc, ())), np.int64, int(off[-1]))
    return dict(post_off=off, post_cluster=ids)


def save(idx: TopKIndex, path, threads: int = 0) -> None:
    """index.save (index.py:122-128): the reference's FOCUSIDX/1 bytes, rendered
    by the native writer (fx_index_write), written to a temp file in the same
    directory and renamed into place."""
    h = idx.header
    V, D = h.vocab, h.dim
    head = "\n".join([_MAGIC, f"stream_id={h.stream_id}", f"D={D}", f"V={V}", f"n={h.n_objects}",
                      format_config(h.config).rstrip("\n"), "[CLUSTERS]"]) + "\n"
    ex = idx.device.export(centroids=True) if idx.device is not None else None
    if idx._clusters is not None or ex is None or "centroids" not in ex:
        ca = _cluster_arrays(idx.clusters.values(), V, D)
    else:
        ca = ex
    pa = _posting_arrays(idx.postings, V) if idx._postings is not None or ex is None else ex
    hb = head.encode("utf-8")
    tmp = f"{path}.tmp.{os.getpid()}"
    try:
        _lib.check(_lib.load().fx_index_write(
            os.fsencode(tmp), hb, len(hb), len(ca["cluster_ids"]), D, V, _lib.p64(ca["cluster_ids"]),
            _lib.pf64(ca["centroids"]), _lib.p64(ca["reps"]), _lib.p64(ca["mem_off"]), _lib.p64(ca["mem_oid"]),
            _lib.p64(ca["mem_fid"]), _lib.p64(ca["cls_off"]), _lib.p32(ca["cls_id"]), _lib.p32(ca["cls_rank"]),
            _lib.p64(pa["post_off"]), _lib.p64(pa["post_cluster"]), int(threads)))
        os.replace(tmp, path)
    finally:
        if os.path.exists(tmp):
            os.unlink(tmp)


_NO_CMID = -(1 << 63)
_HEADER_KEYS = ("stream_id", "D", "V", "n")


def _header_from_lines(text: str) -> IndexHeader:
    """The header block of a FOCUSIDX/1 file (index.py:147-167 semantics: the
    four stream keys, everything else is the config text; KeyError /
    ValueError become DataError, parse_config raises its own DataError)."""
    stream, cfg_lines = {}, []
    for line in text.split("\n") if text else ():
        key, _, value = line.partition("=")
        if key in _HEADER_KEYS:
            stream[key] = value
        else:
            cfg_lines.append(line)
    try:
        vocab = int(stream["V"])
        stream_id, dim, n = stream["stream_id"], int(stream["D"]), int(stream["n"])
        return IndexHeader(stream_id=stream_id, dim=dim, vocab=vocab, n_objects=n,
                           config=parse_config("\n".join(cfg_lines)))
    except (KeyError, ValueError) as exc:
        raise DataError(f"bad index header: {exc}") from exc


def load(path) -> TopKIndex:
    """index.load (index.py:131-204) through the native reader
    (csrc/index_read.cu: CRC-32, line split, multi-threaded record parse into
    CSR arrays, the reference's errors in its order).  Clusters and postings
    are materialised as Python objects only when asked for; lookup and query
    post the arrays on the device directly."""
    L = _lib.load()
    h = _lib.vp()
    _lib.check(L.fx_index_read(os.fsencode(path), ctypes.byref(h)))
    try:
        n = ctypes.c_int64(0)
        _lib.check(L.fx_index_file_header(h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(max(1, n.value))
        _lib.check(L.fx_index_file_header(h, buf, n.value, ctypes.byref(n)))
        header = _header_from_lines(buf.raw[:n.value].decode("utf-8"))
        _lib.check(L.fx_index_file_parse(h, header.vocab))
        sz = np.zeros(7, np.int64)
        _lib.check(L.fx_index_file_sizes(h, _lib.p64(sz)))
        C, ncen, nmem, nfr, ncls, npc, npid = (int(x) for x in sz)
        f = dict(cid=np.empty(C, np.int64), cmid=np.empty(C, np.int64), cen_off=np.empty(C + 1, np.int64),
                 cen=np.empty(ncen, np.float64), mem_off=np.empty(C + 1, np.int64), mem=np.empty(nmem, np.int64),
                 fr_off=np.empty(C + 1, np.int64), fr=np.empty(nfr, np.int64), cls_off=np.empty(C + 1, np.int64),
                 cls=np.empty(ncls, np.int32), rank=np.empty(ncls, np.int32), post_cls=np.empty(npc, np.int32),
                 post_off=np.empty(npc + 1, np.int64), post_ids=np.empty(npid, np.int64))
        _lib.check(L.fx_index_file_export(
            h, _lib.p64(f["cid"]), _lib.p64(f["cmid"]), _lib.p64(f["cen_off"]), _lib.pf64(f["cen"]),
            _lib.p64(f["mem_off"]), _lib.p64(f["mem"]), _lib.p64(f["fr_off"]), _lib.p64(f["fr"]),
            _lib.p64(f["cls_off"]), _lib.p32(f["cls"]), _lib.p32(f["rank"]), _lib.p32(f["post_cls"]),
            _lib.p64(f["post_off"]), _lib.p64(f["post_ids"])))
    finally:
        L.fx_index_file_free(h)
    return TopKIndex(header=header, file_arrays=f)


def _device_from_file(f: dict, header: IndexHeader, device: int | None = None) -> DeviceIndex:
    """Post a loaded file's CSR arrays on the device (clusters in id order).
    The device rebuilds the postings from the class sets (K3); a file whose
    postings disagree with its own class sets is rejected here."""
    V, D, C = header.vocab, header.dim, f["cid"].size
    order = np.argsort(f["cid"], kind="stable")
    ids = np.ascontiguousarray(f["cid"][order])
    mlen = np.diff(f["mem_off"])[order]
    if not np.array_equal(mlen, np.diff(f["fr_off"])[order]):
        raise DataError("cluster member and frame lists differ in length")
    def gather(off, vals, lens):  # segments of `vals` in id order (vectorised)
        o = np.zeros(C + 1, np.int64)
        np.cumsum(lens, out=o[1:])
        idx = np.repeat(off[:-1][order] - o[:-1], lens) + np.arange(int(o[-1]), dtype=np.int64)
        return o, np.ascontiguousarray(vals[idx])
    mem_off, mem = gather(f["mem_off"], f["mem"], mlen)
    _, fr = gather(f["fr_off"], f["fr"], mlen)
    klen = np.diff(f["cls_off"])[order]
    cls_off, cls = gather(f["cls_off"], f["cls"], klen)
    _, rank = gather(f["cls_off"], f["rank"], klen)
    cls = np.ascontiguousarray(np.where(cls == -1, V, cls).astype(np.int32))
    rank = np.ascontiguousarray(rank.astype(np.int32))
    cmid = f["cmid"][order]
    reps = np.ascontiguousarray(np.where(cmid == _NO_CMID, -1, cmid).astype(np.int64))
    cen = None
    clen = np.diff(f["cen_off"])
    if C and np.all(clen == D):
        cen = np.ascontiguousarray(f["cen"].reshape(C, D)[order])
    L = _lib.load()
    h = _lib.vp()
    _lib.check(L.fx_index_build(C, V, header.k, D, _lib.device() if device is None else device, _lib.p64(ids),
                                _lib.pf64(cen) if cen is not None else None, _lib.p64(reps), _lib.p64(mem_off),
                                _lib.p64(mem), _lib.p64(fr), _lib.p64(cls_off), _lib.p32(cls), _lib.p32(rank),
                                ctypes.byref(h)))
    dev = DeviceIndex(h)
    ex = dev.export(centroids=False)
    po, pc = ex["post_off"], ex["post_cluster"]
    fo = f["post_off"]
    for j, c in enumerate(f["post_cls"].tolist()):
        enc = V if c == -1 else c
        if not np.array_equal(pc[po[enc]:po[enc + 1]], f["post_ids"][fo[j]:fo[j + 1]]):
            raise DataError(f"postings of class {c} disagree with the cluster class sets")
    if int(po[-1]) != int(fo[-1]):
        raise DataError("postings disagree with the cluster class sets")
    return dev


__all__ = ["IndexHeader", "TopKIndex", "DeviceIndex", "build", "lookup", "decode_class", "save", "load"]
