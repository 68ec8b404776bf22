"""Parity at the configurations the headline numbers are quoted on.

The device ingest of the bench's own device-generated stream (synth.generate,
the C2 and C3 workloads of BASELINE.json) is compared with the CPU oracle bit
for bit (oracle/scale_parity.py): is_dup, top-K, cluster of every object,
distance_computations, float64 centroid bits, representatives, members,
class ranks, postings.  The C2 prefix is long enough for the B = 4096
steady state (batches are capped at a quarter of the objects seen) and the
Zipf-dominant cluster's long float64 fold chain; the C3 shape crosses the
live-set saturation at L = 20 k (every object seeds; every later batch
evicts through the size-1 FIFO).
"""

import os

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _check(n_gen, n, t, m, seed, batch=0):
    from oracle import scale_parity
    from paper_1801_03493_b200 import synth
    data = synth.generate(n_gen, dim=2048, vocab=1000, n_stream_classes=100, seed=seed)
    torch.cuda.synchronize()
    rep = scale_parity.check_synth(data, n, 4, t, m, 1000, threads=os.cpu_count(), batch=batch)
    del data
    torch.cuda.empty_cache()
    print(rep)
    return rep


@pytest.mark.timeout(900)
def test_c2_prefix_250k_of_bench_stream():
    """First 250 k objects of the bench's 1M-object C2 stream (seed 0):
    ~50 batches at B = 4096, one cluster holding ~60 % of the objects."""
    rep = _check(1_000_000, 250_000, 7.5, 100, seed=0)
    assert rep["mismatches"] == 0, rep["mismatch_by_field"]
    assert rep["classified"] > 190_000


@pytest.mark.timeout(1200)
def test_c3_shape_saturated_live_set_20k():
    """C3 shape at D = 2048: T = 5 (every classified object seeds), M = 20 k,
    40 k objects -> the live set saturates at 20 k and ~12 k evictions
    follow; the TC screen runs many column tiles and CTA waves."""
    rep = _check(40_000, 40_000, 5.0, 20_000, seed=1)
    assert rep["mismatches"] == 0, rep["mismatch_by_field"]
    assert rep["clusters"] > 20_000
