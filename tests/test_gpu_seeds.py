"""Seed-heavy streams (the C3 "small T" shape): most objects seed, probable
seeds are decided in parallel inside a resolve window, together with the
evictions they cause once the live count reaches M (victims taken from the
FIFO of live size-1 clusters; a window is cut where a victim was joined).  The
device ingest must equal the CPU oracle bit for bit: cluster of every
object, distance_computations, float64 centroid bits, representatives."""

import numpy as np
import pytest

from oracle import oracle as O
from oracle import streamgen

pytestmark = pytest.mark.gpu

fx = pytest.importorskip("paper_1801_03493_b200")


def _run(seed, t, m, dim, n=2500, classes=400, batch=0, dup_rate=0.2):
    spec = streamgen.Spec(n_objects=n, dim=dim, vocab=500, n_stream_classes=classes, seed=seed,
                          duplicate_rate=dup_rate)
    st = streamgen.generate(spec)
    prof = O.default_profiles(spec.vocab)["cheap"]
    dup = O.dup_flags(st.fids, st.sigs, 0.01)
    keep = ~dup
    feats = np.zeros((n, dim), np.float32)
    feats[keep] = O.extract_features(prof, seed, st.oids[keep], st.feats[keep]).astype(np.float32)
    k = 4
    topk = np.zeros((n, k), np.int32)
    topk[keep] = O.classify_topk(prof, seed, st.oids[keep], st.true_class[keep], k)
    ref = O.ingest(st.oids, st.fids, st.sigs, feats, topk, k, t, m, is_dup=dup)
    cfg = fx.Config("cheap", k=k, l_s=spec.vocab, t=t, m=m)
    idx, rep, s = fx.ingest_arrays(st.oids, st.fids, st.sigs, feats, cfg, fx.make_default_profiles(500)["cheap"],
                                   vocab=500, seed=seed, true_class=st.true_class.astype(np.int32), batch=batch)
    cl, _, _ = s.object_results(n, k)
    assert np.array_equal(cl.astype(np.int64), ref.cluster_of)
    assert rep.distance_computations == ref.distance_computations
    ex = idx.device.export()
    cen = np.array([cc.centroid for cc in ref.clusters])
    assert np.array_equal(ex["centroids"].view(np.uint64), cen.view(np.uint64))
    assert ex["reps"].tolist() == [cc.centroid_member_id for cc in ref.clusters]
    return rep


@pytest.mark.parametrize("seed,t,m,dim,batch", [
    (31, 0.5, 100000, 64, 0),     # every object seeds, no eviction (C3 before saturation)
    (32, 0.5, 700, 64, 256),      # seeds cross M mid-window: parallel seeds, then evictions
    (33, 0.5, 40, 32, 128),       # saturated from the start: every seed evicts
    (34, 1.4, 100000, 128, 0),    # mixed joins and seeds (classes ~ T)
    (35, 0.0, 100000, 16, 512),   # T = 0: only exact duplicates join
])
def test_seed_heavy_streams_match_oracle(seed, t, m, dim, batch):
    _run(seed, t, m, dim, batch=batch)


@pytest.mark.parametrize("seed,t,m,dim,batch,classes,dup", [
    (36, 1.4, 200, 128, 256, 400, 0.2),   # joins and evictions mixed: joined size-1 clusters cut windows
    (37, 0.5, 300, 64, 512, 400, 0.0),    # no dedup: every seed keeps size 1, FIFO of earlier windows
    (38, 0.5, 300, 64, 512, 400, 0.6),    # heavy dedup: size-1 FIFO drains, seeds evict each other / themselves
    (39, 1.0, 64, 64, 0, 60, 0.3),        # few classes, tiny M: long-lived large clusters never evicted
    (40, 0.5, 1000, 32, 128, 400, 0.2),   # M crossed inside the 8th batch, then every batch evicts
])
def test_window_evictions_match_oracle(seed, t, m, dim, batch, classes, dup):
    _run(seed, t, m, dim, n=4000, classes=classes, batch=batch, dup_rate=dup)


@pytest.mark.timeout(600)
def test_large_saturated_stream_many_cta_waves():
    """30 k objects against up to 5 k live clusters: the TMA screen runs
    several CTA waves over many snapshot column tiles (residuals found by the
    cross-tile row minimum), every batch evicts through the size-1 FIFO."""
    _run(41, 0.5, 5000, 64, n=30000, classes=500, batch=0, dup_rate=0.2)
