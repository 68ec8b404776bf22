"""Generate the golden parity fixtures in tests/golden/ by running the
UNMODIFIED reference (`focusidx`, imported from /root/reference/pkg/src).

Run in the build container (the reference does not exist on the GPU box):

    python tools/gen_golden.py

For every case it
  1. generates the stream with the reference `simharness.generate_stream`
     and checks that oracle/streamgen.py reproduces it bit-for-bit
     (the digests are stored so tests can re-check on any machine);
  2. runs the reference `ingest_stream` with a `classify_fn` that wraps the
     reference `classifiers.classify` and (optionally) rounds the extracted
     feature to float32 -- the GPU path ingests float32 features;
  3. records is_dup, top-K, cluster of every object, every cluster record
     (centroid float64 bits, members, frames, representative, class ranks,
     insertion distances), postings, the IngestReport, and query results
     from the reference `QuerySession` for several classes / k_x / ranges.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from focusidx import classifiers, simharness  # noqa: E402
from focusidx.core import AccuracyTarget, Config, RankedClassification  # noqa: E402
from focusidx.ingest import ingest_stream  # noqa: E402
from focusidx.query import QuerySession  # noqa: E402

from oracle import streamgen  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


CASES = [
    # name, StreamSpec kwargs, Config kwargs, extra
    ("small_d64", dict(n_objects=2000, seed=7, dim=64, vocab=1000, stream_id="small"),
     dict(profile_id="cheap", k=4, l_s=1000, t=1.0, m=20), dict(seed=0, f32=True)),
    ("demo_c1", dict(n_objects=10_000, dim=128, vocab=100, n_stream_classes=100, seed=0),
     dict(profile_id="cheap", k=4, l_s=100, t=1.6, m=100), dict(seed=0, f32=True)),
    ("evict_d32", dict(n_objects=3000, dim=32, vocab=50, n_stream_classes=50, seed=3),
     dict(profile_id="cheap", k=3, l_s=50, t=0.45, m=30), dict(seed=5, f32=True)),
    ("f64_d16", dict(n_objects=1500, dim=16, vocab=200, n_stream_classes=40, seed=11),
     dict(profile_id="cheap", k=5, l_s=200, t=0.6, m=10), dict(seed=2, f32=False)),
    ("nodiff_d24", dict(n_objects=1200, dim=24, vocab=300, n_stream_classes=30, seed=4),
     dict(profile_id="cheap", k=2, l_s=300, t=0.7, m=15), dict(seed=1, f32=True, pixel_eps=-1.0)),
    ("spec_d32", dict(n_objects=2000, dim=32, vocab=500, n_stream_classes=60, seed=9),
     dict(profile_id="cheap+spec6", k=3, l_s=6, t=0.8, m=25), dict(seed=4, f32=True, specialize=6)),
    ("gt_d8", dict(n_objects=800, dim=8, vocab=50, n_stream_classes=20, seed=2),
     dict(profile_id="gt", k=1, l_s=50, t=0.3, m=40), dict(seed=0, f32=True)),
    ("c2_prefix_d2048", dict(n_objects=3000, dim=2048, vocab=1000, n_stream_classes=100, seed=0),
     dict(profile_id="cheap", k=4, l_s=1000, t=7.5, m=100), dict(seed=0, f32=True)),
    ("c3_shape_d2048", dict(n_objects=1500, dim=2048, vocab=1000, n_stream_classes=100, seed=1),
     dict(profile_id="cheap", k=4, l_s=1000, t=5.0, m=400), dict(seed=0, f32=True)),
]


def row_hash(a) -> np.ndarray:
    """First 8 bytes (little-endian u64) of sha256 of each row's float64 bytes."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return np.array([int.from_bytes(hashlib.sha256(r.tobytes()).digest()[:8], "little")
                     for r in a], dtype=np.uint64)


def csr(lists, dtype):
    off = np.zeros(len(lists) + 1, dtype=np.int64)
    for i, l in enumerate(lists):
        off[i + 1] = off[i] + len(l)
    vals = np.array([x for l in lists for x in l], dtype=dtype)
    return off, vals


def run_case(name, spec_kw, cfg_kw, extra):
    spec = simharness.StreamSpec(**spec_kw)
    header, objects = simharness.generate_stream(spec)
    mine = streamgen.generate(streamgen.Spec(**spec_kw))
    n = len(objects)
    ref_oids = np.array([o.object_id for o in objects], dtype=np.int64)
    ref_fids = np.array([o.frame_id for o in objects], dtype=np.int64)
    ref_sigs = np.array([o.pixel_signature for o in objects]).reshape(n, spec.sig_dim)
    ref_feats = np.array([o.feature for o in objects]).reshape(n, spec.dim)
    ref_tc = np.array([o.true_class for o in objects], dtype=np.int64)
    assert np.array_equal(ref_oids, mine.oids) and np.array_equal(ref_fids, mine.fids)
    assert np.array_equal(ref_sigs, mine.sigs) and np.array_equal(ref_feats, mine.feats)
    assert np.array_equal(ref_tc, mine.true_class), name
    in_digest = digest(ref_oids, ref_fids, ref_sigs, ref_feats, ref_tc)

    profiles = classifiers.make_default_profiles(spec.vocab)
    if extra.get("specialize"):
        hist = {}
        for o in objects:
            hist[o.true_class] = hist.get(o.true_class, 0) + 1
        sp = classifiers.specialize_profile(profiles["cheap"], hist, extra["specialize"])
        profiles[sp.profile_id] = sp
    cfg = Config(targets=AccuracyTarget(), **cfg_kw)
    profile = profiles[cfg.profile_id]
    seed = extra["seed"]
    f32 = extra["f32"]
    eps = extra.get("pixel_eps", 0.01)

    log = {}

    def classify_fn(prof, obj, s):
        rc = classifiers.classify(prof, obj, s)
        feat = rc.feature.astype(np.float32) if f32 else rc.feature
        log[obj.object_id] = (rc.top(cfg.k).classes(), feat)
        return RankedClassification(rc.ranked, feat)

    idx, rep = ingest_stream(header, objects, cfg, profiles, pixel_eps=eps, seed=seed,
                             classify_fn=classify_fn)
    is_dup = np.array([o.object_id not in log for o in objects], dtype=bool)
    topk = np.zeros((n, cfg.k), dtype=np.int32)
    feats_used = np.zeros((n, spec.dim), dtype=np.float32 if f32 else np.float64)
    for i, o in enumerate(objects):
        if o.object_id in log:
            topk[i] = log[o.object_id][0]
            feats_used[i] = log[o.object_id][1]
    cluster_of = np.full(n, -1, dtype=np.int64)
    cids = sorted(idx.clusters)
    for cid in cids:
        for oid in idx.clusters[cid].member_object_ids:
            cluster_of[oid] = cid
    cl = [idx.clusters[c] for c in cids]
    mem_off, mem_oid = csr([c.member_object_ids for c in cl], np.int64)
    _, mem_fid = csr([c.frame_ids for c in cl], np.int64)
    ins_off, ins_val = csr([c.insertion_distances for c in cl], np.float64)
    cr_off, cr_cls = csr([list(c.class_best_rank.keys()) for c in cl], np.int32)
    _, cr_rank = csr([list(c.class_best_rank.values()) for c in cl], np.int32)
    cent = np.array([c.centroid for c in cl]).reshape(len(cl), spec.dim)
    reps = np.array([-1 if c.centroid_member_id is None else c.centroid_member_id for c in cl],
                    dtype=np.int64)
    post_cls = sorted(idx.postings)
    po_off, po_ids = csr([idx.postings[c] for c in post_cls], np.int64)

    # queries: the most frequent true classes and a couple of absent ones
    counts = np.bincount(ref_tc, minlength=spec.vocab)
    top_classes = list(np.argsort(-counts, kind="stable")[:6])
    qclasses = [int(c) for c in top_classes] + [int(np.argmin(counts))]
    fmax = int(ref_fids.max()) if n else 0
    ranges = [None, (fmax // 4, fmax // 2)]
    q_rows, q_fr, q_ob = [], [], []
    gt = profiles["gt"]
    objmap = {o.object_id: o for o in objects}
    for qc in qclasses:
        for kx in sorted({1, max(1, cfg.k // 2), cfg.k}):
            for ri, tr in enumerate(ranges):
                sess = QuerySession(idx, gt, objmap, ingest_profile=profile)
                res = sess.route_query(qc, k_x=kx, time_range=tr)
                q_rows.append([qc, kx, ri, res.gt_inferences, res.clusters_examined,
                               res.clusters_matched, len(res.frame_ids), len(res.object_ids)])
                q_fr.append(list(res.frame_ids))
                q_ob.append(list(res.object_ids))
    qf_off, qf_val = csr(q_fr, np.int64)
    qo_off, qo_val = csr(q_ob, np.int64)

    out = dict(
        name=name, spec_kw=repr(spec_kw), cfg_kw=repr(cfg_kw), extra=repr(extra),
        input_digest=in_digest, feats_digest=digest(feats_used[~is_dup]),
        is_dup=is_dup, topk=topk, cluster_of=cluster_of,
        cl_ids=np.array(cids, dtype=np.int64), cl_rep=reps, cl_centroid_h64=row_hash(cent),
        mem_off=mem_off, mem_oid=mem_oid, mem_fid=mem_fid, ins_off=ins_off, ins_val=ins_val,
        cr_off=cr_off, cr_cls=cr_cls, cr_rank=cr_rank,
        post_cls=np.array(post_cls, dtype=np.int64), po_off=po_off, po_ids=po_ids,
        report=np.array([rep.objects_seen, rep.objects_classified, rep.clusters_emitted,
                         rep.distance_computations, rep.gt_invocations], dtype=np.int64),
        report_cost=np.array([rep.ingest_cost_units, rep.dedup_savings_units]),
        q_rows=np.array(q_rows, dtype=np.int64), q_ranges=np.array(
            [[-1, -1], list(ranges[1])], dtype=np.int64),
        qf_off=qf_off, qf_val=qf_val, qo_off=qo_off, qo_val=qo_val,
    )
    if cent.size <= 400_000:
        out["cl_centroid"] = cent
    if extra.get("specialize"):
        out["class_set"] = np.array(profile.class_set, dtype=np.int64)
        out["spec_rho"] = np.array([profile.rank_model.rho, profile.rank_model.p1, profile.cost_units])
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: n={n} classified={rep.objects_classified} clusters={rep.clusters_emitted} "
          f"dc={rep.distance_computations} -> {os.path.getsize(path) / 1e3:.0f} KB")


def rank_vectors():
    """Known-answer vectors for the rank draw and the first uniform of
    default_rng([seed, oid, w]) (classifiers.py:126-133)."""
    rng = np.random.default_rng(123)
    seeds = rng.integers(0, 2**40, 300)
    oids = rng.integers(0, 2**35, 300)
    oids[:100] = rng.integers(0, 10**6, 100)
    words = rng.integers(0, 2, 300)
    u = np.array([np.random.default_rng([int(s), int(o), int(w)]).random()
                  for s, o, w in zip(seeds, oids, words)])
    m = classifiers.RankModel(0.7, 0.95)
    us = np.concatenate([u, rng.random(2000), 1 - rng.random(200) * 1e-6])
    rk = np.array([m.rank_from_uniform(float(x), 1000) for x in us], dtype=np.int64)
    m2 = classifiers.RankModel(0.3, 0.5)
    rk2 = np.array([m2.rank_from_uniform(float(x), 7) for x in us], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "rank_vectors.npz"), seeds=seeds, oids=oids,
                        words=words, u=u, us=us, rank_07_095_1000=rk, rank_03_05_7=rk2)
    print("rank_vectors written")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    only = sys.argv[1:]
    rank_vectors()
    for case in CASES:
        if not only or case[0] in only:
            run_case(*case)
