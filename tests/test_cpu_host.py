"""CPU-only checks of the host side: the C ABI library loads and exports every
symbol include/focus_b200.h declares (no compute calls), and the per-profile
device tables reproduce the reference classifier exactly (the K1a kernel's
splice emulated in numpy, checked against the oracle / golden vectors)."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
import golden_util as GU

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(REPO, "include", "focus_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fx_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_1801_03493_b200 import _build, _lib
    _build.build()
    lib = ctypes.CDLL(_build.LIB)
    names = _header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    # the ctypes binding covers the header exactly
    assert set(_lib.EXPORTED) == set(names)
    L = _lib.load()
    assert L.fx_version() == 1


def test_package_imports_without_gpu():
    import paper_1801_03493_b200 as fx
    assert fx.OTHER_CLASS == -1
    assert fx.make_default_profiles(10)["cheap"].output_length == 10


def _emulate_k1a(profile, seed, oids, tcls, k):
    """numpy emulation of k_rank_topk (csrc/ingest.cu) on the host tables."""
    from paper_1801_03493_b200 import classifiers as C
    thr, emit, fill = C.device_tables(profile, seed, k)
    fill = fill.reshape(-1, k)
    out = np.zeros((len(oids), k), np.int32)
    V = profile.vocab
    for i, (o, c) in enumerate(zip(oids, tcls)):
        if profile.kind == C.GROUND_TRUTH:
            rank = 1
        else:
            u = int(O.first_u64([seed, int(o), 0])) >> 11
            rank = 1 + int(np.sum(thr <= np.uint64(u)))
        e = int(emit[c])
        row = fill[e]
        out[i] = [row[j] if j < rank - 1 else (e if j == rank - 1 else row[j - 1]) for j in range(k)]
    out[out == V] = -1
    return out


@pytest.mark.parametrize("name", GU.case_names())
def test_device_tables_reproduce_reference_topk(name):
    import paper_1801_03493_b200 as fx
    c = GU.load(name)
    g = c.g
    p = c.profile
    if p.class_set is not None:
        prof = fx.ClassifierProfile(p.profile_id, fx.SPECIALIZED, p.vocab, fx.RankModel(p.p1, p.rho), p.cost_units,
                                    p.feature_noise_sigma, p.class_set)
    else:
        prof = fx.make_default_profiles(p.vocab)[c.cfg["profile_id"]]
    keep = ~g["is_dup"]
    got = _emulate_k1a(prof, c.extra["seed"], c.stream.oids[keep], c.stream.true_class[keep], c.cfg["k"])
    assert np.array_equal(got, g["topk"][keep])


def test_rank_thresholds_match_rank_model():
    from paper_1801_03493_b200 import classifiers as C
    rng = np.random.default_rng(1)
    for p1, rho, out_len, k in [(0.7, 0.95, 1000, 8), (0.3, 0.5, 7, 6), (0.7, 0.76, 6, 4), (0.99, 0.0, 50, 3),
                                (1.0, 0.0, 10, 2)]:
        thr = np.array(C.rank_thresholds(p1, rho, out_len, k), dtype=np.uint64)
        us = np.concatenate([rng.integers(0, 1 << 53, 4000, dtype=np.int64).astype(np.uint64),
                             thr[thr < np.uint64(1 << 53)], thr[thr < np.uint64(1 << 53)] - np.uint64(1)])
        for u in us.tolist():
            r = O.rank_from_uniform(u * (1.0 / 9007199254740992.0), p1, rho, out_len)
            dev = 1 + int(np.sum(thr <= np.uint64(u)))
            assert min(r, k + 1) == dev, (p1, rho, u)


def test_error_taxonomy_mirrors_reference():
    from paper_1801_03493_b200 import errors as E
    assert issubclass(E.MissingTrueClass, E.DataError)
    assert issubclass(E.KxTooLarge, E.UsageError)
    assert issubclass(E.DimensionMismatch, E.DataError)
    assert E.STATUS[50] is E.KxTooLarge and E.STATUS[20] is E.MissingTrueClass
