"""The tcgen05 TF32 screen kernel: values against a float64 reference and the
rigorous error bound the ingest relies on (|v - d^2| <= 2 gamma |a||b|)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
fx = pytest.importorskip("paper_1801_03493_b200")
from paper_1801_03493_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("na,nb,dim", [(128, 128, 32), (300, 100, 2048), (77, 200, 128), (512, 1000, 64),
                                       (130, 129, 4)])
def test_tc_screen_matches_float64_within_bound(na, nb, dim):
    rng = np.random.default_rng(na + nb + dim)
    means = rng.standard_normal((20, dim))
    A = (means[rng.integers(0, 20, na)] + 0.11 * rng.standard_normal((na, dim))).astype(np.float32)
    B = (means[rng.integers(0, 20, nb)] + 0.02 * rng.standard_normal((nb, dim))).astype(np.float32)
    out = np.empty((na, nb), np.float32)
    _lib.check(_lib.load().fx_debug_screen_tc(0, na, nb, dim, _lib.pv(A), _lib.pv(B), _lib.pv(out)))
    a64, b64 = A.astype(np.float64), B.astype(np.float64)
    ref = ((a64[:, None, :] - b64[None, :, :]) ** 2).sum(-1)
    gam = 2.0 ** -9 + dim * 2.0 ** -22
    bound = 2 * gam * np.linalg.norm(a64, axis=1)[:, None] * np.linalg.norm(b64, axis=1)[None, :] + 1e-3
    err = np.abs(out.astype(np.float64) - ref)
    assert np.all(err <= bound), float((err / bound).max())
    # and it really is a tensor-core GEMM, not garbage: typical error far below the bound
    assert np.median(err / bound) < 0.2


@pytest.mark.parametrize("na,nb,dim", [(1000, 300, 2048), (130, 7, 200), (77, 129, 64), (4096, 101, 2048),
                                       (20000, 1000, 256), (6000, 800, 2048)])  # last two: several CTA waves
def test_tma_and_cp_async_staging_bit_identical(na, nb, dim, monkeypatch):
    """TMA tiled boxes (SWIZZLE_128B) and the cp.async fallback stage the same
    operands in the same K order: the screen values must agree bit for bit."""
    rng = np.random.default_rng(7 * na + dim)
    A = rng.standard_normal((na, dim)).astype(np.float32)
    B = rng.standard_normal((nb, dim)).astype(np.float32)
    outs = {}
    for mode in ("cp", "tma"):
        monkeypatch.setenv("FOCUS_B200_TCLOAD", mode)
        out = np.empty((na, nb), np.float32)
        _lib.check(_lib.load().fx_debug_screen_tc(0, na, nb, dim, _lib.pv(A), _lib.pv(B), _lib.pv(out)))
        outs[mode] = out
    assert np.array_equal(outs["cp"].view(np.uint32), outs["tma"].view(np.uint32))
