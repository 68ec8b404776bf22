"""GPU parity: the CUDA path (through the C ABI) against the reference's own
golden outputs (tests/golden/, produced by tools/gen_golden.py) and against
the CPU oracle at other sizes.  Integer / index / byte results bit-exact;
float64 centroids bit-exact (exact float64 paths in numpy order)."""

import numpy as np
import pytest

from oracle import oracle as O
from oracle import streamgen
import golden_util as GU

pytestmark = pytest.mark.gpu

fx = pytest.importorskip("paper_1801_03493_b200")


def _profile(c):
    p = c.profile
    if p.class_set is not None:
        return fx.ClassifierProfile(p.profile_id, fx.SPECIALIZED, p.vocab, fx.RankModel(p.p1, p.rho), p.cost_units,
                                    p.feature_noise_sigma, p.class_set)
    return fx.make_default_profiles(p.vocab)[c.cfg["profile_id"]]


def _cfg(c):
    d = c.cfg
    return fx.Config(d["profile_id"], k=d["k"], l_s=d["l_s"], t=d["t"], m=d["m"])


def _run_case(c, batch=0, compact=False):
    st = c.stream
    feats = c.feats
    if compact:
        feats = feats[~c.g["is_dup"]]
    return fx.ingest_arrays(st.oids, st.fids, st.sigs, feats, _cfg(c), _profile(c), vocab=c.spec.vocab,
                            seed=c.extra["seed"], pixel_eps=c.pixel_eps, true_class=st.true_class.astype(np.int32),
                            compact=compact, batch=batch)


def _check_against_golden(c, idx, rep, stream):
    g = c.g
    n, k = c.spec.n_objects, c.cfg["k"]
    cl, dup, tk = stream.object_results(n, k)
    assert np.array_equal(dup, g["is_dup"]), "is_dup"
    keep = ~dup
    V = c.spec.vocab
    tk = tk.copy()
    tk[tk == V] = -1
    assert np.array_equal(tk[keep], g["topk"][keep]), "top-K"
    assert np.array_equal(cl.astype(np.int64), g["cluster_of"]), "cluster assignment"
    r = g["report"]
    assert (rep.objects_seen, rep.objects_classified, rep.clusters_emitted, rep.distance_computations) == \
        tuple(int(x) for x in r[:4])
    ex = idx.device.export()
    exp = GU.golden_clusters(g)
    assert ex["cluster_ids"].tolist() == [e["cluster_id"] for e in exp]
    for i, e in enumerate(exp):
        a, b = ex["mem_off"][i], ex["mem_off"][i + 1]
        assert ex["mem_oid"][a:b].tolist() == e["members"], ("members", i)
        assert ex["mem_fid"][a:b].tolist() == e["frames"], ("frames", i)
        assert int(ex["reps"][i]) == e["rep"], ("rep", i)
        ca, cb = ex["cls_off"][i], ex["cls_off"][i + 1]
        ranks = {(-1 if x == V else x): y for x, y in zip(ex["cls_id"][ca:cb].tolist(), ex["cls_rank"][ca:cb].tolist())}
        assert ranks == e["ranks"], ("class ranks", i)
    assert np.array_equal(GU.row_hash(ex["centroids"]), g["cl_centroid_h64"]), "centroid float64 bits"
    assert idx.postings == GU.golden_postings(g)


@pytest.mark.parametrize("name", GU.case_names())
def test_ingest_matches_reference_golden(name):
    c = GU.load(name)
    idx, rep, stream = _run_case(c)
    _check_against_golden(c, idx, rep, stream)


@pytest.mark.parametrize("name", ["small_d64", "evict_d32", "f64_d16"])
@pytest.mark.parametrize("batch", [64, 320])
def test_ingest_batch_size_invariance(name, batch):
    c = GU.load(name)
    idx, rep, stream = _run_case(c, batch=batch, compact=(batch == 64))
    _check_against_golden(c, idx, rep, stream)


@pytest.mark.parametrize("name", ["small_d64", "evict_d32", "f64_d16", "c2_prefix_d2048"])
def test_pinned_host_inputs(name):
    """Pinned host inputs (the e2e bench's case): chunked asynchronous H2D on a
    side stream overlapped with the ingest of earlier chunks."""
    import torch
    c = GU.load(name)

    def pinned(a):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        return t

    st = c.stream
    keep = [pinned(np.ascontiguousarray(x)) for x in (st.oids, st.fids, st.sigs, c.feats,
                                                      st.true_class.astype(np.int32))]
    oids, fids, sigs, feats, tcls = (t.numpy() for t in keep)
    idx, rep, stream = fx.ingest_arrays(oids, fids, sigs, feats, _cfg(c), _profile(c), vocab=c.spec.vocab,
                                        seed=c.extra["seed"], pixel_eps=c.pixel_eps, true_class=tcls)
    _check_against_golden(c, idx, rep, stream)


@pytest.mark.parametrize("name", GU.case_names())
def test_queries_match_reference_golden(name):
    c = GU.load(name)
    idx, rep, stream = _run_case(c)
    labels = {int(o): int(t) for o, t in zip(c.stream.oids, c.stream.true_class)}
    gt = fx.make_default_profiles(c.spec.vocab)["gt"]
    for qc, kx, tr, exp in GU.golden_queries(c.g):
        sess = fx.QuerySession(idx, gt, None, ingest_profile=_profile(c), labels=labels)
        got = sess.route_query(qc, k_x=kx, time_range=tr)
        for key, val in exp.items():
            assert getattr(got, key) == val, (name, qc, kx, tr, key)


def test_chunked_ingest_equals_single_call():
    """Streams fed in several fx_ingest calls (chunk boundaries inside dedup
    runs) give the same index as one call."""
    c = GU.load("small_d64")
    st = c.stream
    cfg, prof = _cfg(c), _profile(c)
    s = fx.ingest.Stream(c.spec.dim, c.spec.sig_dim, c.spec.vocab, cfg.k, cfg.t, cfg.m, c.pixel_eps, 0, None, 128)
    s.set_rank_model(prof, c.extra["seed"])
    cuts = [0, 7, 8, 500, 1001, 1002, 1999, 2000]
    for a, b in zip(cuts, cuts[1:]):
        s.ingest(st.oids[a:b].copy(), st.fids[a:b].copy(), np.ascontiguousarray(st.sigs[a:b]),
                 np.ascontiguousarray(c.feats[a:b]), true_class=st.true_class[a:b].astype(np.int32))
    dix, rep = s.finalize()
    idx = fx.TopKIndex(fx.IndexHeader("s", c.spec.dim, c.spec.vocab, c.spec.n_objects, cfg), device=dix)
    _check_against_golden(c, idx, rep, s)


def test_dropin_ingest_stream_with_classify_fn():
    """The reference-facing API on DetectedObjects with a classify_fn plugin
    (the reference's own call convention, ingest.py:52-61)."""
    c = GU.load("demo_c1")
    st = c.stream
    prof = _profile(c)
    objs = [fx.DetectedObject(int(o), int(f), 0.0, st.sigs[i], st.feats[i], int(t))
            for i, (o, f, t) in enumerate(zip(st.oids, st.fids, st.true_class))]
    k = c.cfg["k"]
    topk_rows = {int(o): row for o, row, d in zip(st.oids, c.g["topk"], c.g["is_dup"]) if not d}
    feat_rows = {int(o): c.feats[i] for i, o in enumerate(st.oids)}
    calls = []

    def classify_fn(profile, obj, seed):
        calls.append(obj.object_id)
        ranked = tuple((int(x), 0.9) for x in topk_rows[obj.object_id])
        return fx.RankedClassification(ranked, feat_rows[obj.object_id])

    header = fx.StreamHeader("demo", 30.0, c.spec.dim, c.spec.sig_dim, c.spec.vocab)
    idx, rep = fx.ingest_stream(header, objs, _cfg(c), {prof.profile_id: prof}, seed=c.extra["seed"],
                                classify_fn=classify_fn)
    assert calls == [int(o) for o, d in zip(st.oids, c.g["is_dup"]) if not d]
    assert rep.distance_computations == int(c.g["report"][3])
    assert rep.clusters_emitted == int(c.g["report"][2])
    assert idx.postings == GU.golden_postings(c.g)
    exp = GU.golden_clusters(c.g)
    for e in exp:
        got = idx.clusters[e["cluster_id"]]
        assert got.member_object_ids == e["members"]
        assert got.centroid_member_id == e["rep"]


@pytest.mark.parametrize("seed,t,m,dim", [(21, 1.2, 7, 16), (22, 0.0, 50, 8), (23, 3.0, 3, 40), (24, 0.35, 200, 24)])
def test_random_configs_match_oracle(seed, t, m, dim):
    spec = streamgen.Spec(n_objects=1500, dim=dim, vocab=60, n_stream_classes=25, seed=seed)
    st = streamgen.generate(spec)
    prof = O.default_profiles(spec.vocab)["cheap"]
    dup = O.dup_flags(st.fids, st.sigs, 0.01)
    keep = ~dup
    feats = np.zeros((spec.n_objects, dim), np.float32)
    feats[keep] = O.extract_features(prof, seed, st.oids[keep], st.feats[keep]).astype(np.float32)
    k = 3
    topk = np.zeros((spec.n_objects, k), np.int32)
    topk[keep] = O.classify_topk(prof, seed, st.oids[keep], st.true_class[keep], k)
    ref = O.ingest(st.oids, st.fids, st.sigs, feats, topk, k, t, m, is_dup=dup)
    cfg = fx.Config("cheap", k=k, l_s=spec.vocab, t=t, m=m)
    idx, rep, s = fx.ingest_arrays(st.oids, st.fids, st.sigs, feats, cfg, fx.make_default_profiles(60)["cheap"],
                                   vocab=60, seed=seed, true_class=st.true_class.astype(np.int32), batch=192)
    cl, _, _ = s.object_results(spec.n_objects, k)
    assert np.array_equal(cl.astype(np.int64), ref.cluster_of)
    assert rep.distance_computations == ref.distance_computations
    ex = idx.device.export()
    cen = np.array([cc.centroid for cc in ref.clusters])
    assert np.array_equal(ex["centroids"].view(np.uint64), cen.view(np.uint64))
    assert ex["reps"].tolist() == [cc.centroid_member_id for cc in ref.clusters]


@pytest.mark.parametrize("name", ["small_d64", "spec_d32", "gt_d8", "f64_d16"])
def test_saved_index_file_equals_reference_file(name, tmp_path):
    """Device ingest -> fx.save: the FOCUSIDX/1 bytes the reference's
    index.save wrote for the same stream (tests/golden/index_<case>.focusidx)."""
    import os
    c = GU.load(name)
    golden = os.path.join(GU.GOLDEN, f"index_{name}.focusidx")
    with open(golden, "rb") as fh:
        want = fh.read()
    stream_id = want.split(b"\n")[1].decode().partition("=")[2]
    st = c.stream
    idx, rep, _ = fx.ingest_arrays(st.oids, st.fids, st.sigs, c.feats, _cfg(c), _profile(c), vocab=c.spec.vocab,
                                   seed=c.extra["seed"], pixel_eps=c.pixel_eps,
                                   true_class=st.true_class.astype(np.int32), stream_id=stream_id)
    out = tmp_path / "idx.focusidx"
    fx.save(idx, str(out))
    assert out.read_bytes() == want


def test_lookup_on_loaded_index_file():
    """fx.load (reference parser) then fx.lookup: the device index is posted on
    first lookup; every class x k_x equals the filter of the file's class ranks."""
    import os
    path = os.path.join(GU.GOLDEN, "index_spec_d32.focusidx")
    idx = fx.load(path)
    V = idx.header.vocab
    for cls in list(range(V)) + [fx.OTHER_CLASS]:
        for kx in range(1, idx.header.k + 1):
            want = sorted(cid for cid, c in idx.clusters.items() if c.class_best_rank.get(cls, 10 ** 9) <= kx)
            assert fx.lookup(idx, cls, kx) == want, (cls, kx)
