"""CPU: the feature-noise restatement the device runs (csrc/noise.cu) against
the real libraries -- numpy's Generator.standard_normal (extract_feature,
reference classifiers.py:152-158) and glibc's log1p."""
import math

import numpy as np
import pytest

from oracle import ziggurat as Z


def test_header_tables_are_numpys():
    import glob
    import os
    (so,) = glob.glob(os.path.join(os.path.dirname(np.__file__), "random", "_generator*.so"))
    b = open(so, "rb").read()
    o = b.find((0x000EF33D8025EF6A).to_bytes(8, "little"))
    ki, wi, fi = Z.header_tables()
    assert np.array_equal(ki, np.frombuffer(b[o:o + 2048], "<u8"))
    assert np.array_equal(wi.view(np.uint64), np.frombuffer(b[o - 2048:o], "<u8"))
    assert np.array_equal(fi.view(np.uint64), np.frombuffer(b[o - 4096:o - 2048], "<u8"))


@pytest.mark.parametrize("seed", [0, 7, 2**40 + 3])
def test_ziggurat_equals_standard_normal(seed):
    tables = Z.header_tables()
    slow = 0
    for oid in list(range(40)) + [2**33 + 5, 2**63 - 1]:
        ss = [seed, oid, 1]
        want = np.random.default_rng(ss).standard_normal(2048)
        raw = np.random.PCG64(np.random.SeedSequence(ss)).random_raw(4200)
        got = Z.normals(raw, 2048, tables, log1p=Z.glibc_log1p)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), oid


def test_glibc_log1p_restatement():
    rng = np.random.default_rng(3)
    u = np.concatenate([rng.random(20000), rng.random(3000) * 1e-6, 1 - rng.random(3000) * 1e-6,
                        rng.random(3000) * 0.6, rng.random(500) * 2.0**-40, np.array([0.0, 0.5, 0.2928932])])
    # next_double values: k * 2^-53
    u = np.floor(u * 2.0**53) / 2.0**53
    bad = [float(v) for v in u if Z.glibc_log1p(-float(v)) != math.log1p(-float(v))]
    assert not bad, bad[:5]
