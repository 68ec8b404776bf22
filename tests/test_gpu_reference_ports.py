"""The reference's own unit scenarios (pkg/tests/test_clustering.py,
test_ingest.py, test_index.py, test_query.py) run against the device path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fx = pytest.importorskip("paper_1801_03493_b200")


def _cluster_run(features, t, m, topk=None, sigs=None, fids=None, eps=-1.0, k=1, vocab=20, oids=None):
    F = np.asarray(features, np.float64)
    n, d = F.shape
    oids = np.arange(n, dtype=np.int64) if oids is None else np.asarray(oids, np.int64)
    fids = oids.copy() if fids is None else np.asarray(fids, np.int64)
    sigs = np.repeat(oids[:, None].astype(np.float64), 4, axis=1) if sigs is None else np.asarray(sigs, np.float64)
    if topk is None:
        topk = np.zeros((n, k), np.int32)
    cfg = fx.Config("cheap", k=k, l_s=vocab, t=t, m=m)
    prof = fx.make_default_profiles(vocab)["cheap"]
    idx, rep, s = fx.ingest_arrays(oids, fids, sigs, F, cfg, prof, vocab=vocab, topk=np.asarray(topk, np.int32),
                                   pixel_eps=eps)
    cl, dup, _ = s.object_results(n, k)
    return idx, rep, cl


def test_threshold_join_and_eviction_scenario():
    # test_clustering.py:18-41
    idx, rep, cl = _cluster_run([[0, 0, 0], [0.5, 0, 0], [5, 5, 5], [0.2, 0.2, 0], [9, 9, 9]], t=1.0, m=2)
    assert cl.tolist() == [0, 0, 1, 0, 2]
    assert rep.distance_computations == 6
    c = idx.clusters
    assert sorted(c) == [0, 1, 2]
    assert c[0].member_object_ids == [0, 1, 3]
    np.testing.assert_allclose(c[0].centroid, [0.7 / 3, 0.2 / 3, 0.0])
    assert c[0].centroid_member_id == 3
    assert c[1].centroid_member_id == 2


def test_t_zero_keeps_singletons():
    _, rep, _ = _cluster_run([[float(i)] for i in range(5)], t=0.0, m=100)
    assert rep.clusters_emitted == 5


def test_exact_match_joins_at_t_zero():
    _, _, cl = _cluster_run([[1.0], [1.0]], t=0.0, m=10)
    assert cl.tolist() == [0, 0]


def test_centroid_running_mean_and_dedup_member():
    # object 2 is a pixel-diff duplicate of object 1: member without feature
    sigs = [[0.0] * 4, [10.0] * 4, [10.0] * 4]
    idx, rep, cl = _cluster_run([[0.0], [3.0], [99.0]], t=10.0, m=5, sigs=sigs, fids=[0, 1, 2], eps=0.01)
    assert rep.objects_classified == 2
    c = idx.clusters[0]
    np.testing.assert_allclose(c.centroid, [1.5])
    assert c.member_object_ids == [0, 1, 2]


def test_representative_tie_breaks_to_smaller_object_id():
    idx, _, _ = _cluster_run([[0.0], [2.0]], t=10.0, m=5, oids=[4, 9])
    assert idx.clusters[0].centroid_member_id == 4


def test_class_best_rank_keeps_minimum():
    idx, _, _ = _cluster_run([[0.0], [0.1]], t=10.0, m=5, topk=[[7, 8], [8, 7]], k=2)
    assert idx.clusters[0].class_best_rank == {7: 1, 8: 1}


def test_ingest_dedup_scenario():
    # test_ingest.py:34-65
    P = lambda oid, frame, sig: fx.DetectedObject(oid, frame, 0.0, np.array(sig, float),  # noqa: E731
                                                  np.array([float(oid), 0.0]), 3)
    objs = [P(0, 0, [0.0, 0.0]), P(1, 1, [0.0, 0.0]), P(2, 2, [10.0, 10.0]), P(3, 3, [10.005, 10.005]),
            P(4, 5, [10.005, 10.005]), P(5, 6, [20.0, 20.0])]
    header = fx.StreamHeader("t", 30.0, 2, 2, 1000)
    cfg = fx.Config("cheap", k=8, l_s=1000, t=0.0, m=100)
    profiles = fx.make_default_profiles(1000)
    idx, rep = fx.ingest_stream(header, objs, cfg, profiles)
    assert (rep.objects_seen, rep.objects_classified, rep.clusters_emitted) == (6, 4, 4)
    assert rep.ingest_cost_units == pytest.approx(4 * 58.0 / 8)
    assert sorted(c.member_object_ids for c in idx.clusters.values()) == [[0, 1], [2, 3], [4], [5]]
    _, rep2 = fx.ingest_stream(header, objs, cfg, profiles, pixel_eps=-1.0)
    assert rep2.objects_classified == 6


def test_pixel_diff_thresholds():
    # test_ingest.py:17-31
    o = lambda oid, frame, sig: fx.DetectedObject(oid, frame, 0.0, np.array(sig, float), np.zeros(2), 3)  # noqa
    a = o(0, 0, [0.0, 0.0])
    assert fx.pixel_diff(a, o(1, 1, [0.0, 0.0]), 0.01)
    assert fx.pixel_diff(a, o(1, 1, [0.01, 0.01]), 0.01)
    assert not fx.pixel_diff(a, o(1, 1, [0.011, 0.011]), 0.01)
    assert fx.pixel_diff(a, o(1, 0, [0.0, 0.0]), 0.01)
    assert not fx.pixel_diff(a, o(1, 2, [0.0, 0.0]), 0.01)
    assert not fx.pixel_diff(a, o(1, 1, [0.0, 0.0]), -1.0)
    with pytest.raises(fx.SignatureLengthMismatch):
        fx.pixel_diff(a, o(1, 1, [0.0]), 0.01)


def _hand_index(k=4):
    def cl(cid, ranks, members, rep=None):
        return fx.Cluster(cluster_id=cid, centroid=np.zeros(2), member_object_ids=list(members),
                          frame_ids=[m * 2 for m in members], class_best_rank=dict(ranks),
                          centroid_member_id=members[0] if rep is None else rep, sealed=True)
    cfg = fx.Config("cheap", k=k, l_s=50, t=0.25, m=100)
    header = fx.IndexHeader(stream_id="s", dim=2, vocab=50, n_objects=6, config=cfg)
    return fx.build([cl(0, {7: 1, 9: 3}, (0, 1)), cl(1, {9: 1, fx.OTHER_CLASS: 2}, (2,)),
                     cl(2, {7: 4, fx.OTHER_CLASS: 1}, (3, 4, 5))], header)


def test_build_postings_and_lookup():
    # test_index.py:38-63
    idx = _hand_index()
    assert idx.postings == {7: [0, 2], 9: [0, 1], fx.OTHER_CLASS: [1, 2]}
    assert fx.lookup(idx, 7) == [0, 2]
    assert fx.lookup(idx, 7, k_x=3) == [0]
    assert fx.lookup(idx, 9, k_x=2) == [1]
    assert fx.lookup(idx, 9, k_x=4) == [0, 1]
    assert fx.lookup(idx, 42) == []
    with pytest.raises(fx.KxTooLarge):
        fx.lookup(idx, 7, k_x=5)
    with pytest.raises(fx.KxTooLarge):
        fx.lookup(idx, 7, k_x=0)


def test_build_rejects_duplicate_ids():
    cfg = fx.Config("cheap", k=4, l_s=50, t=0.25, m=100)
    header = fx.IndexHeader(stream_id="s", dim=2, vocab=50, n_objects=2, config=cfg)
    c = lambda cid, r: fx.Cluster(cid, np.zeros(2), [cid], [cid], {r: 1}, cid, True)  # noqa: E731
    with pytest.raises(fx.DuplicateClusterId):
        fx.build([c(1, 3), c(1, 4)], header)


_TRUE = {0: 7, 1: 7, 2: 9, 3: 12, 4: 12, 5: 12}


@pytest.fixture()
def session():
    profiles = fx.make_default_profiles(1000)
    spec = fx.specialize_profile(profiles["cheap"], {7: 5, 9: 4}, l_s=2)
    objects = {o: fx.DetectedObject(o, o * 2, 0.0, np.zeros(4), np.zeros(2), c) for o, c in _TRUE.items()}
    return fx.QuerySession(_hand_index(), profiles["gt"], objects, ingest_profile=spec)


def test_verification_rejects_impostors(session):
    # test_query.py:50-58
    res = session.execute_query(fx.QueryRequest(7))
    assert (res.clusters_examined, res.clusters_matched) == (2, 1)
    assert res.object_ids == (0, 1) and res.frame_ids == (0, 2)
    assert res.gt_inferences == 2 and res.query_cost_units == pytest.approx(116.0)


def test_memoization(session):
    first = session.execute_query(fx.QueryRequest(7))
    again = session.execute_query(fx.QueryRequest(7))
    assert again.object_ids == first.object_ids and again.gt_inferences == 0
    assert session.execute_query(fx.QueryRequest(9)).gt_inferences == 1
    assert session.gt_inferences_total() == 3


def test_kx_and_time_range(session):
    assert session.execute_query(fx.QueryRequest(7, k_x=3)).clusters_examined == 1
    res = session.execute_query(fx.QueryRequest(7, time_range=(0, 1)))
    assert res.frame_ids == (0,) and res.object_ids == (0,) and res.clusters_matched == 1


def test_unknown_class(session):
    with pytest.raises(fx.UnknownClass):
        session.execute_query(fx.QueryRequest(60))
    with pytest.raises(fx.UnknownClass):
        session.execute_query(fx.QueryRequest(-2))


def test_other_routing(session):
    res = session.route_query(12)
    assert res.object_ids == (3, 4, 5) and res.clusters_examined == 2 and res.clusters_matched == 1
    assert session.route_query(7).object_ids == (0, 1)
    res = session.query_other(13)
    assert res.object_ids == () and res.clusters_examined == 2 and res.clusters_matched == 0
    assert session.execute_query(fx.QueryRequest(fx.OTHER_CLASS)).object_ids == (3, 4, 5)


def test_other_requires_specialized_profile():
    profiles = fx.make_default_profiles(1000)
    objects = {o: fx.DetectedObject(o, o * 2, 0.0, np.zeros(4), np.zeros(2), c) for o, c in _TRUE.items()}
    plain = fx.QuerySession(_hand_index(), profiles["gt"], objects, ingest_profile=profiles["cheap"])
    with pytest.raises(fx.UnknownClass):
        plain.execute_query(fx.QueryRequest(fx.OTHER_CLASS))
    with pytest.raises(fx.UnknownClass):
        plain.query_other(12)


def test_batched_query(session):
    batches = list(session.batched_query(fx.QueryRequest(7), [1, 3, 4]))
    assert batches[0].object_ids == (0, 1)
    assert batches[1].clusters_examined == 0
    assert batches[2].clusters_examined == 1 and batches[2].object_ids == ()
    total = sum(b.gt_inferences for b in batches)
    profiles = fx.make_default_profiles(1000)
    spec = fx.specialize_profile(profiles["cheap"], {7: 5, 9: 4}, l_s=2)
    objects = {o: fx.DetectedObject(o, o * 2, 0.0, np.zeros(4), np.zeros(2), c) for o, c in _TRUE.items()}
    single = fx.QuerySession(_hand_index(), profiles["gt"], objects, ingest_profile=spec)
    assert total == single.execute_query(fx.QueryRequest(7, k_x=4)).gt_inferences
    with pytest.raises(fx.NonMonotoneSchedule):
        list(session.batched_query(fx.QueryRequest(7), [2, 2]))


def test_missing_true_class_raised_on_touch():
    profiles = fx.make_default_profiles(1000)
    objects = {o: fx.DetectedObject(o, o * 2, 0.0, np.zeros(4), np.zeros(2), None if o == 2 else c)
               for o, c in _TRUE.items()}
    s = fx.QuerySession(_hand_index(), profiles["gt"], objects)
    assert s.execute_query(fx.QueryRequest(7)).object_ids == (0, 1)  # rep 2 untouched
    with pytest.raises(fx.MissingTrueClass):
        s.execute_query(fx.QueryRequest(9))
