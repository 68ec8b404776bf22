"""K1b FC head oracle (CPU): the float64 restatement ranks like a brute-force
sort, and -- when the reference is importable here -- the reference pipeline
driven by the oracle head as its classify_fn produces exactly the oracle
ingest on the oracle head's top-K (pins the oracle FC path to the reference)."""

import os
import sys

import numpy as np
import pytest

from oracle import oracle as O
from oracle import streamgen


def test_fc_topk_matches_bruteforce():
    rng = np.random.default_rng(3)
    F = rng.standard_normal((200, 24)).astype(np.float32)
    W = rng.standard_normal((37, 24)).astype(np.float32)
    b = rng.standard_normal(37).astype(np.float32)
    top, flag = O.fc_topk(F, W, b, 5)
    L = F.astype(np.float64) @ W.astype(np.float64).T + b.astype(np.float64)
    for i in range(F.shape[0]):
        ref = sorted(range(37), key=lambda c: (-L[i, c], c))[:5]
        assert top[i].tolist() == ref
    assert not flag.any()


def test_fc_topk_ties_go_to_smaller_id_and_are_flagged():
    W = np.array([[1.0, 0.0], [1.0, 0.0], [0.0, 1.0]], np.float32)
    F = np.array([[2.0, 1.0]], np.float32)
    top, flag = O.fc_topk(F, W, None, 2)
    assert top[0].tolist() == [0, 1] and flag[0]


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_reference_pipeline_with_oracle_head_equals_oracle_ingest():
    sys.path.insert(0, REF)
    try:
        from focusidx import core, ingest
    finally:
        sys.path.remove(REF)
    spec = streamgen.Spec(n_objects=600, dim=32, vocab=50, n_stream_classes=20, seed=8)
    st = streamgen.generate(spec)
    rng = np.random.default_rng(11)
    W = rng.standard_normal((50, 32)).astype(np.float32)
    b = (0.1 * rng.standard_normal(50)).astype(np.float32)
    feats = st.feats.astype(np.float32)
    objs = [core.DetectedObject(int(o), int(f), f / 30.0, s.astype(np.float64), x, int(c))
            for o, f, s, x, c in zip(st.oids, st.fids, st.sigs, feats, st.true_class)]
    from focusidx import streamio
    header = streamio.StreamHeader("fc", 30.0, 32, st.sigs.shape[1], 50)
    from focusidx import classifiers as RC
    profiles = RC.make_default_profiles(50)
    cfg = core.Config("cheap", k=4, l_s=50, t=2.5, m=15)
    k = cfg.k

    def cfn(profile, obj, seed):
        return O.fc_classify_fn(W, b)(profile, obj, seed)

    idx, rep = ingest.ingest_stream(header, objs, cfg, profiles, classify_fn=cfn)
    dup = O.dup_flags(st.fids, st.sigs, 0.01)
    top, _ = O.fc_topk(feats, W, b, k)
    res = O.ingest(st.oids, st.fids, st.sigs, feats, top, k, cfg.t, cfg.m, is_dup=dup)
    assert rep.distance_computations == res.distance_computations
    assert len(idx.clusters) == len(res.clusters)
    for a, c in zip([idx.clusters[i] for i in sorted(idx.clusters)], res.clusters):
        assert a.member_object_ids == c.member_object_ids
        assert a.class_best_rank == {int(x): int(y) for x, y in c.class_best_rank.items()}
