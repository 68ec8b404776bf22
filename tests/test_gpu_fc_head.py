"""K1b FC classifier head on the device (tcgen05 TF32 screen of the logits +
float64 re-score of the candidates) against the float64 oracle head.
Top-K classes must be bit-exact for every object neither side flags as within
the float64 logit margin (the north star's stated exception); ingest driven
by the head must equal the oracle ingest on the oracle head's top-K."""

import numpy as np
import pytest

from oracle import oracle as O
from oracle import streamgen

pytestmark = pytest.mark.gpu

fx = pytest.importorskip("paper_1801_03493_b200")


def _feats(n, dim, seed):
    st = streamgen.generate(streamgen.Spec(n_objects=n, dim=dim, vocab=1000, n_stream_classes=50, seed=seed))
    return st, st.feats.astype(np.float32)


@pytest.mark.parametrize("n,dim,V,k,seed", [(3000, 2048, 1000, 4, 0), (2000, 64, 100, 8, 1), (1500, 128, 300, 1, 2),
                                            (700, 256, 17, 16, 3)])
def test_topk_matches_float64_oracle(n, dim, V, k, seed):
    _, F = _feats(n, dim, seed)
    rng = np.random.default_rng(100 + seed)
    W = (rng.standard_normal((V, dim)) / np.sqrt(dim)).astype(np.float32)
    b = (0.1 * rng.standard_normal(V)).astype(np.float32)
    head = fx.FCHead(W, b)
    tk, conf, flag = head.topk(F, k)
    ref, rflag = O.fc_topk(F, W, b, k)
    ok = ~(flag | rflag)
    assert ok.mean() > 0.99
    assert np.array_equal(tk[ok], ref[ok])
    # confidences: softmax of the emitted logits, descending
    L = O.fc_logits(F, W, b)
    p = np.exp(L - L.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    np.testing.assert_allclose(conf[ok], np.take_along_axis(p, ref.astype(np.int64), axis=1)[ok], rtol=1e-2, atol=1e-6)


@pytest.mark.parametrize("n,dim,V,k,seed", [(70000, 64, 1000, 4, 5), (40000, 128, 300, 2, 6)])
def test_persistent_logits_many_tiles_per_cta(n, dim, V, k, seed):
    # >= 3 (object, class) tiles per CTA of the persistent k_fc_tcp (both TMEM
    # accumulators reused, phases wrapping), a partial last class tile, and
    # (n > 65536) two object chunks of the head
    rng = np.random.default_rng(200 + seed)
    F = rng.standard_normal((n, dim)).astype(np.float32)
    W = (rng.standard_normal((V, dim)) / np.sqrt(dim)).astype(np.float32)
    b = (0.1 * rng.standard_normal(V)).astype(np.float32)
    tk, conf, flag = fx.FCHead(W, b).topk(F, k)
    ref, rflag = O.fc_topk(F, W, b, k)
    ok = ~(flag | rflag)
    assert ok.mean() > 0.99
    assert np.array_equal(tk[ok], ref[ok])


def test_near_ties_use_the_all_class_rescore_and_stay_exact():
    # duplicated weight rows (+ tiny perturbations) put many classes inside the
    # TF32 error band of the K-th logit: the kernel must fall back to scoring
    # every class in float64
    _, F = _feats(600, 128, 5)
    rng = np.random.default_rng(9)
    base = rng.standard_normal((8, 128)).astype(np.float32)
    W = np.repeat(base, 40, axis=0) + (1e-6 * rng.standard_normal((320, 128))).astype(np.float32)
    head = fx.FCHead(W, None)
    tk, _, flag = head.topk(F, 4)
    ref, rflag = O.fc_topk(F, W, None, 4)
    ok = ~(flag | rflag)
    assert ok.sum() > 100
    assert np.array_equal(tk[ok], ref[ok])


def test_ingest_with_fc_head_equals_oracle_ingest():
    spec = streamgen.Spec(n_objects=3000, dim=64, vocab=200, n_stream_classes=30, seed=5)
    st = streamgen.generate(spec)
    F = st.feats.astype(np.float32)
    rng = np.random.default_rng(4)
    W = (rng.standard_normal((200, 64)) / 8.0).astype(np.float32)
    b = (0.05 * rng.standard_normal(200)).astype(np.float32)
    k, t, m = 4, 0.9, 25
    dup = O.dup_flags(st.fids, st.sigs, 0.01)
    ref_top, rflag = O.fc_topk(F, W, b, k)
    topk = np.where(dup[:, None], 0, ref_top).astype(np.int32)
    ref = O.ingest(st.oids, st.fids, st.sigs, F, topk, k, t, m, is_dup=dup)
    cfg = fx.Config("cheap", k=k, l_s=200, t=t, m=m)
    prof = fx.make_default_profiles(200)["cheap"]
    idx, rep, stream = fx.ingest_arrays(st.oids, st.fids, st.sigs, F, cfg, prof, vocab=200, fc_head=fx.FCHead(W, b))
    cl, isdup, tk = stream.object_results(spec.n_objects, k)
    assert not rflag[~dup].any()
    assert np.array_equal(isdup, dup)
    assert np.array_equal(tk[~dup], ref_top[~dup])
    assert np.array_equal(cl.astype(np.int64), ref.cluster_of)
    assert rep.distance_computations == ref.distance_computations
    assert stream.counters()["fc_flagged"] == 0
    assert idx.postings == O.build_postings(ref.clusters)
