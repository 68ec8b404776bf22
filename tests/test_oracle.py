"""Pin the CPU oracle against the reference's own outputs (tests/golden/) and
against numpy for the third-party primitives it restates.  CPU only."""

import os

import numpy as np
import pytest

from oracle import oracle as O
import golden_util as GU


@pytest.mark.parametrize("n", list(range(0, 140)) + [255, 256, 257, 1000, 2048, 4097, 8192, 8193,
                                                      20000, 70001])
def test_pairwise_sum_matches_numpy(n):
    rng = np.random.default_rng(n)
    a = rng.random(n) * 10.0 ** rng.integers(-3, 5)
    assert O.pairwise_sum(a) == np.add.reduce(a)
    x = rng.standard_normal((2, n))
    f = rng.standard_normal(n).astype(np.float32)
    ref = np.linalg.norm(x - f, axis=1)
    d = x - f.astype(np.float64)
    assert np.array_equal(ref, np.sqrt([O.pairwise_sum(r * r) for r in d]))


def test_mean_matches_numpy():
    rng = np.random.default_rng(0)
    for s in (1, 2, 3, 7, 8, 9, 16, 17, 33):
        for _ in range(40):
            a, b = rng.standard_normal(s), rng.standard_normal(s)
            assert O.pairwise_sum(np.abs(a - b)) / s == float(np.mean(np.abs(a - b)))


def test_first_uniform_matches_reference_vectors():
    g = np.load(os.path.join(GU.GOLDEN, "rank_vectors.npz"))
    got = np.array([O.first_uniform(int(s), int(o), int(w))
                    for s, o, w in zip(g["seeds"], g["oids"], g["words"])])
    assert np.array_equal(got, g["u"])


def test_first_u64_matches_numpy():
    for ints in ([0], [1], [0, 0, 0], [5, 2**33, 7, 9, 11], [2**63, 1], [7, 0xA110]):
        assert O.first_u64(ints) == np.random.default_rng(ints).bit_generator.random_raw()


def test_rank_from_uniform_matches_reference_vectors():
    g = np.load(os.path.join(GU.GOLDEN, "rank_vectors.npz"))
    r1 = [O.rank_from_uniform(float(u), 0.7, 0.95, 1000) for u in g["us"]]
    r2 = [O.rank_from_uniform(float(u), 0.3, 0.5, 7) for u in g["us"]]
    assert np.array_equal(r1, g["rank_07_095_1000"])
    assert np.array_equal(r2, g["rank_03_05_7"])


def test_rank_frozen_values():
    # test_classifiers.py:33-40 frozen values
    assert O.rank_from_uniform(0.2, 0.7, 0.95, 1000) == 1
    assert O.rank_from_uniform(0.7, 0.7, 0.95, 1000) == 1
    assert O.rank_from_uniform(0.8, 0.7, 0.95, 1000) == 9
    assert O.rank_from_uniform(0.999, 0.7, 0.95, 1000) == 113
    assert O.rank_from_uniform(0.999, 0.7, 0.95, 50) == 50


@pytest.mark.parametrize("name", GU.case_names())
def test_oracle_ingest_matches_reference(name):
    c = GU.load(name)
    g = c.g
    st = c.stream
    dup = O.dup_flags(st.fids, st.sigs, c.pixel_eps)
    assert np.array_equal(dup, g["is_dup"])
    k = c.cfg["k"]
    topk = np.zeros((c.spec.n_objects, k), dtype=np.int32)
    topk[~dup] = O.classify_topk(c.profile, c.extra["seed"], st.oids[~dup], st.true_class[~dup], k)
    assert np.array_equal(topk, g["topk"])
    res = O.ingest(st.oids, st.fids, st.sigs, c.feats, topk, k, c.cfg["t"], c.cfg["m"],
                   c.pixel_eps, is_dup=dup)
    assert np.array_equal(res.cluster_of, g["cluster_of"])
    assert res.distance_computations == int(g["report"][3])
    assert len(res.clusters) == int(g["report"][2])
    exp = GU.golden_clusters(g)
    for mine, ref in zip(res.clusters, exp):
        assert mine.cluster_id == ref["cluster_id"]
        assert mine.member_object_ids == ref["members"]
        assert mine.frame_ids == ref["frames"]
        assert (mine.centroid_member_id if mine.centroid_member_id is not None else -1) == ref["rep"]
        assert mine.class_best_rank == ref["ranks"]
        assert np.array_equal(np.asarray(mine.insertion_distances), ref["ins"])
    cents = np.array([cl.centroid for cl in res.clusters]).reshape(len(res.clusters), c.spec.dim)
    assert np.array_equal(GU.row_hash(cents), g["cl_centroid_h64"])
    if "cl_centroid" in g:
        assert np.array_equal(cents.view(np.uint64), g["cl_centroid"].view(np.uint64))
    assert O.build_postings(res.clusters) == GU.golden_postings(g)


@pytest.mark.parametrize("name", GU.case_names())
def test_oracle_queries_match_reference(name):
    c = GU.load(name)
    g = c.g
    clusters = [O.OracleCluster(d["cluster_id"], None, d["members"], d["frames"], d["ranks"],
                                None if d["rep"] < 0 else d["rep"]) for d in GU.golden_clusters(g)]
    gt = {int(o): int(t) for o, t in zip(c.stream.oids, c.stream.true_class)}
    for qc, kx, tr, exp in GU.golden_queries(g):
        sess = O.OracleSession(clusters, c.cfg["k"], c.spec.vocab, gt, ingest_profile=c.profile)
        got = sess.route_query(qc, kx, tr)
        for key, val in exp.items():
            assert got[key] == val, (name, qc, kx, tr, key)
