"""Load a golden case (tests/golden/*.npz, written by tools/gen_golden.py from
the reference) and rebuild its inputs with the oracle's stream generator."""

from __future__ import annotations

import ast
import glob
import hashlib
import os
from dataclasses import dataclass

import numpy as np

from oracle import oracle as O
from oracle import streamgen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not p.endswith("rank_vectors.npz"))


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def row_hash(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return np.array([int.from_bytes(hashlib.sha256(r.tobytes()).digest()[:8], "little")
                     for r in a], dtype=np.uint64)


@dataclass
class Case:
    name: str
    g: dict
    spec: streamgen.Spec
    cfg: dict
    extra: dict
    stream: streamgen.Stream
    profile: O.Profile
    profiles: dict
    feats: np.ndarray      # features the ingest clusters (f32 or f64), dup rows zero
    pixel_eps: float


_cache = {}


def load(name: str) -> Case:
    if name in _cache:
        return _cache[name]
    g = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    spec_kw = ast.literal_eval(str(g["spec_kw"]))
    cfg = ast.literal_eval(str(g["cfg_kw"]))
    extra = ast.literal_eval(str(g["extra"]))
    spec = streamgen.Spec(**spec_kw)
    st = streamgen.generate(spec)
    assert digest(st.oids, st.fids, st.sigs, st.feats, st.true_class) == str(g["input_digest"]), \
        "stream generator no longer reproduces the reference stream"
    profiles = O.default_profiles(spec.vocab)
    if "class_set" in g:
        rho, p1, cost = (float(x) for x in g["spec_rho"])
        cs = tuple(int(x) for x in g["class_set"])
        profiles[cfg["profile_id"]] = O.Profile(cfg["profile_id"], O.SPECIALIZED, spec.vocab, p1, rho,
                                                cost, 0.05, cs)
    prof = profiles[cfg["profile_id"]]
    is_dup = g["is_dup"]
    ext = O.extract_features(prof, extra["seed"], st.oids[~is_dup], st.feats[~is_dup])
    dt = np.float32 if extra["f32"] else np.float64
    feats = np.zeros((spec.n_objects, spec.dim), dtype=dt)
    feats[~is_dup] = ext.astype(dt)
    assert digest(feats[~is_dup]) == str(g["feats_digest"])
    c = Case(name, g, spec, cfg, extra, st, prof, profiles, feats, extra.get("pixel_eps", 0.01))
    _cache[name] = c
    return c


def golden_clusters(g):
    """Per-cluster dicts from the CSR arrays."""
    out = []
    for i, cid in enumerate(g["cl_ids"].tolist()):
        a, b = g["mem_off"][i], g["mem_off"][i + 1]
        ca, cb = g["cr_off"][i], g["cr_off"][i + 1]
        ia, ib = g["ins_off"][i], g["ins_off"][i + 1]
        out.append(dict(
            cluster_id=cid, members=g["mem_oid"][a:b].tolist(), frames=g["mem_fid"][a:b].tolist(),
            rep=int(g["cl_rep"][i]), ranks=dict(zip(g["cr_cls"][ca:cb].tolist(),
                                                     g["cr_rank"][ca:cb].tolist())),
            ins=g["ins_val"][ia:ib]))
    return out


def golden_postings(g):
    out = {}
    for i, c in enumerate(g["post_cls"].tolist()):
        out[c] = g["po_ids"][g["po_off"][i]:g["po_off"][i + 1]].tolist()
    return out


def golden_queries(g):
    """[(class, k_x, time_range, expected dict)]"""
    rows = []
    ranges = [None, tuple(int(x) for x in g["q_ranges"][1])]
    for j, r in enumerate(g["q_rows"].tolist()):
        qc, kx, ri, gti, ex, ma, nf, no = r
        fr = tuple(g["qf_val"][g["qf_off"][j]:g["qf_off"][j + 1]].tolist())
        ob = tuple(g["qo_val"][g["qo_off"][j]:g["qo_off"][j + 1]].tolist())
        rows.append((qc, kx, ranges[ri], dict(frame_ids=fr, object_ids=ob, gt_inferences=gti,
                                              clusters_examined=ex, clusters_matched=ma)))
    return rows
