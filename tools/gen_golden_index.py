"""Golden FOCUSIDX/1 files written by the UNMODIFIED
reference `focusidx.index.save`, for tests/test_index_files.py and the GPU
round trip in tests/test_gpu_parity.py.  Run in the build container (the
reference does not exist on the GPU box):

    python tools/gen_golden_index.py

  * index_<case>.focusidx: the reference ingest of a golden case
    (tools/gen_golden.py CASES, same classify_fn) saved by the reference;
  * index_edge.focusidx + index_edge.json: a hand-built index whose
    centroids exercise %.9g (exponents, -0, subnormals, 9-digit rounding),
    a cluster without representative, an empty class set and OTHER postings;
    the JSON carries the exact float64 centroids (float.hex) and postings.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "tools"))

from focusidx import classifiers, index, simharness  # noqa: E402
from focusidx.clustering import Cluster  # noqa: E402
from focusidx.core import OTHER_CLASS, AccuracyTarget, Config, RankedClassification  # noqa: E402
from focusidx.ingest import ingest_stream  # noqa: E402

from gen_golden import CASES  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")
FILE_CASES = ("small_d64", "spec_d32", "gt_d8", "f64_d16")


def ingest_case(name, spec_kw, cfg_kw, extra):
    spec = simharness.StreamSpec(**spec_kw)
    header, objects = simharness.generate_stream(spec)
    profiles = classifiers.make_default_profiles(spec.vocab)
    if extra.get("specialize"):
        hist = {}
        for o in objects:
            hist[o.true_class] = hist.get(o.true_class, 0) + 1
        sp = classifiers.specialize_profile(profiles["cheap"], hist, extra["specialize"])
        profiles[sp.profile_id] = sp
    cfg = Config(targets=AccuracyTarget(), **cfg_kw)

    def classify_fn(prof, obj, s):
        rc = classifiers.classify(prof, obj, s)
        feat = rc.feature.astype(np.float32) if extra["f32"] else rc.feature
        return RankedClassification(rc.ranked, feat)

    idx, _ = ingest_stream(header, objects, cfg, profiles, pixel_eps=extra.get("pixel_eps", 0.01),
                           seed=extra["seed"], classify_fn=classify_fn)
    return idx


EDGE_VALUES = [0.0, -0.0, 1e-5, -1.5e-7, 0.1, 1.0 / 3.0, 2.0 / 3.0, 123456789.0, 1234567890.0, 123456789012.0,
               1e16, 100000.0, 5e-324, 2.2250738585072014e-308, 9.9999999949999e-5, 0.99999999951,
               -7.25, 3.14159265358979, 1e-300, 6.02214076e23]


def edge_index():
    from focusidx.index import IndexHeader, build
    D = len(EDGE_VALUES)
    rng = np.random.default_rng(5)
    clusters = []
    specs = [
        (3, 17, [17, 18, 40], [2, 2, 9], {0: 1, 5: 2, OTHER_CLASS: 3}),
        (0, None, [4], [1], {}),
        (11, 100, [100, 101], [30, 31], {OTHER_CLASS: 1}),
        (7, 55, [55], [20], {5: 1, 2: 4}),
    ]
    for j, (cid, rep, mem, frames, ranks) in enumerate(specs):
        cen = np.array(EDGE_VALUES, dtype=np.float64) * (1.0 if j == 0 else rng.uniform(-3, 3))
        clusters.append(Cluster(cluster_id=cid, centroid=cen, member_object_ids=mem, frame_ids=frames,
                                class_best_rank=ranks, centroid_member_id=rep, sealed=True))
    cfg = Config(profile_id="cheap", k=4, l_s=8, t=0.5, m=10, targets=AccuracyTarget())
    header = IndexHeader(stream_id="edge-cam", dim=D, vocab=8, n_objects=200, config=cfg)
    idx = build(clusters, header)
    desc = dict(
        header=dict(stream_id=header.stream_id, dim=D, vocab=8, n_objects=200,
                    config=dict(profile_id="cheap", k=4, l_s=8, t=0.5, m=10)),
        clusters=[dict(cluster_id=c.cluster_id, rep=c.centroid_member_id,
                       centroid=[float(x).hex() for x in c.centroid], members=c.member_object_ids,
                       frames=c.frame_ids, ranks=[[k, v] for k, v in c.class_best_rank.items()])
                  for c in clusters],
        postings=[[k, v] for k, v in idx.postings.items()])
    return idx, desc


if __name__ == "__main__":
    for name, spec_kw, cfg_kw, extra in CASES:
        if name not in FILE_CASES:
            continue
        idx = ingest_case(name, spec_kw, cfg_kw, extra)
        path = os.path.join(OUT, f"index_{name}.focusidx")
        index.save(idx, path)
        print(name, os.path.getsize(path), "bytes")
    idx, desc = edge_index()
    index.save(idx, os.path.join(OUT, "index_edge.focusidx"))
    with open(os.path.join(OUT, "index_edge.json"), "w") as fh:
        json.dump(desc, fh, indent=1)
    print("edge written")
