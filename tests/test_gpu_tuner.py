"""Tuner grid evaluation on the device: the drop-in
GridEvaluator against the reference's own cached evaluator _GridEvaluator
(tuner.py:169-293) on reference-generated samples -- every grid point of
two_step_search must evaluate to the identical ConfigEvaluation (the
reference's contract, test_tuner.py:117-129: the cached path equals running
ingest + query config by config).  The reference runs from baseline/_ref
(pip-installed there, travels with the snapshot); skipped without it."""

import os
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg(c):
    return (c.profile_id, c.k, c.l_s, c.t, c.m, c.targets.precision_target, c.targets.recall_target)


def _ev(e):
    return (_cfg(e.cfg), e.est_recall, e.est_precision, e.ingest_cost, e.query_cost, e.viable)


def _ref():
    for p in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "focusidx")) and p not in sys.path:
            sys.path.append(p)
    try:
        from focusidx import simharness, tuner  # noqa: F401
        return simharness, tuner
    except Exception:
        pytest.skip("reference package not available")


@pytest.mark.timeout(900)
@pytest.mark.parametrize("n,seed,dim", [(700, 11, 64), (2500, 3, 64), (1200, 5, 128)])
def test_grid_equals_reference_evaluator(n, seed, dim):
    sim, rt = _ref()
    import paper_1801_03493_b200 as fx
    from focusidx.classifiers import make_default_profiles
    from focusidx.core import AccuracyTarget
    header, objects = sim.generate_stream(sim.StreamSpec(n_objects=n, n_stream_classes=12, vocab=100, seed=seed,
                                                         dim=dim, stream_id="t"))
    profiles = make_default_profiles(100)
    sample = rt.sample_stream(objects, header.fps, seed=seed)
    targets = AccuracyTarget()
    t_values = rt.derive_t_values(sample)
    cands = rt.candidate_profiles(profiles, sample, (5, 10), True)
    ref = rt._GridEvaluator(header, sample, profiles, targets, 0.01, seed, 100)
    dev = fx.tuner.GridEvaluator(header, sample, profiles, targets, 0.01, seed, 100)
    checked = 0
    for p in cands:
        for k in (1, 2, 4, 8):
            if k > p.output_length:
                continue
            for t in t_values[::3]:
                a, b = ref.evaluate(p, k, t), dev.evaluate(p, k, t)
                assert (a.est_recall, a.est_precision, a.ingest_cost, a.query_cost, a.viable) == \
                       (b.est_recall, b.est_precision, b.ingest_cost, b.query_cost, b.viable), (p.profile_id, k, t)
                assert _cfg(a.cfg) == _cfg(b.cfg)
                checked += 1
    assert checked > 20


@pytest.mark.timeout(900)
def test_two_step_search_with_device_evaluator():
    """two_step_search (the reference's own search) with the device evaluator
    switched in returns the reference's result."""
    sim, rt = _ref()
    import paper_1801_03493_b200 as fx
    from focusidx.classifiers import make_default_profiles
    header, objects = sim.generate_stream(sim.StreamSpec(n_objects=700, n_stream_classes=12, vocab=100, seed=11,
                                                         stream_id="tiny"))
    grid = rt.TuneGrid(k_values=(1, 2, 4, 8), l_s_values=(5, 10))
    want = rt.two_step_search(header, objects, make_default_profiles(100), grid=grid)
    orig = rt._GridEvaluator
    rt._GridEvaluator = fx.tuner.GridEvaluator
    try:
        got = rt.two_step_search(header, objects, make_default_profiles(100), grid=grid)
    finally:
        rt._GridEvaluator = orig
    assert [_ev(e) for e in got.evaluations] == [_ev(e) for e in want.evaluations]
    assert [_ev(e) for e in got.viable] == [_ev(e) for e in want.viable]
