"""Device feature noise (csrc/noise.cu) against numpy:
extract_feature (reference classifiers.py:152-158) is
    feature + sigma * default_rng([seed, oid, 1]).standard_normal(D)
and the device result must be bit-identical (float64), including the
ziggurat's slow paths (u-layer rejections, the idx-0 tail's log1p)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fx = pytest.importorskip("paper_1801_03493_b200")
from paper_1801_03493_b200 import classifiers  # noqa: E402


def _want(F, oids, sigma, seed):
    return np.stack([F[i] + sigma * np.random.default_rng([seed, int(o), 1]).standard_normal(F.shape[1])
                     for i, o in enumerate(oids)])


@pytest.mark.parametrize("D,dtype,seed", [(2048, np.float32, 0), (2048, np.float64, 7), (128, np.float32, 2**40 + 1),
                                          (37, np.float64, 3), (1, np.float32, 5), (33, np.float32, 11)])
def test_extract_features_bit_exact(D, dtype, seed):
    rng = np.random.default_rng(D + seed % 97)
    n = 400
    oids = np.concatenate([np.arange(n - 3), [2**32 - 1, 2**33 + 7, 2**62 + 11]]).astype(np.int64)
    F = rng.standard_normal((n, D)).astype(dtype)
    prof = fx.make_default_profiles(100)["cheap"]
    got = classifiers.extract_features(prof, oids, F, seed)
    want = _want(F, oids, prof.feature_noise_sigma, seed)
    assert got.dtype == np.float64
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_extract_features_many_slow_paths():
    # 12k objects x 2048 normals: ~370k u-layer tests, ~6k idx-0 tail draws
    n, D, seed = 12000, 2048, 123
    rng = np.random.default_rng(9)
    oids = np.sort(rng.choice(10**9, n, replace=False)).astype(np.int64)
    F = np.zeros((n, D), np.float32)
    L = fx._lib.load()
    out = np.empty((n, D), np.float64)
    nflag = np.zeros(1, np.int64)
    fx._lib.check(L.fx_extract_features(fx._lib.device(), n, D, fx._lib.p64(oids), fx._lib.pv(F), fx._lib.FX_F32,
                                        1.0, seed, fx._lib.pf64(out), fx._lib.p64(nflag)))
    for i in range(0, n, 1):
        want = np.random.default_rng([seed, int(oids[i]), 1]).standard_normal(D)
        if not np.array_equal(out[i].view(np.uint64), want.view(np.uint64)):
            j = int(np.flatnonzero(out[i] != want)[0])
            raise AssertionError(f"object {i} (oid {oids[i]}): first difference at normal {j}: "
                                 f"{out[i, j]!r} vs {want[j]!r}")
    assert nflag[0] == 0


def test_sigma_zero_copies():
    prof = fx.make_default_profiles(100)["gt"]
    F = np.random.default_rng(1).standard_normal((50, 64))
    got = classifiers.extract_features(prof, np.arange(50), F, 0)
    assert np.array_equal(got, F)


def test_ingest_stream_device_noise_matches_host_noise():
    """The drop-in's engine-side noise stage == clustering the host-extracted
    features (the reference's extract_feature) -- same clusters, centroids,
    postings and report."""
    from oracle import streamgen
    spec = streamgen.Spec(n_objects=3000, dim=256, vocab=50, n_stream_classes=20, seed=4)
    st = streamgen.generate(spec)
    prof = fx.make_default_profiles(spec.vocab)["cheap"]
    cfg = fx.Config("cheap", k=4, l_s=spec.vocab, t=1.6, m=40)
    dup = fx.ingest.dup_flags(st.fids, st.sigs, 0.01)
    keep = np.flatnonzero(~dup)
    raw = st.feats[keep].astype(np.float64)
    ext = _want(raw, st.oids[keep], prof.feature_noise_sigma, 0)
    tc = st.true_class.astype(np.int32)
    ix1, rep1, s1 = fx.ingest_arrays(st.oids, st.fids, st.sigs, raw, cfg, prof, vocab=spec.vocab, seed=0,
                                     true_class=tc, compact=True, raw_features=True)
    ix2, rep2, s2 = fx.ingest_arrays(st.oids, st.fids, st.sigs, ext, cfg, prof, vocab=spec.vocab, seed=0,
                                     true_class=tc, compact=True)
    assert rep1 == rep2
    assert s1.counters()["noise_flagged"] == 0
    e1, e2 = ix1.device.export(), ix2.device.export()
    for k in e2:
        assert np.array_equal(np.asarray(e1[k]), np.asarray(e2[k])), k
