"""Several engines on one GPU in SM partitions (CUDA green contexts,
fx_device_set_partitions): two engines ingest different streams
concurrently, each in its own partition, and each result equals the CPU
oracle bit for bit (oracle/scale_parity.py)."""

import ctypes
import os
import threading

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_two_engines_in_two_partitions_match_oracle():
    import paper_1801_03493_b200 as fx
    from oracle import scale_parity as SP
    from paper_1801_03493_b200 import _lib, synth
    L = _lib.load()
    sms = ctypes.c_int32(0)
    _lib.check(L.fx_device_set_partitions(0, 2, ctypes.byref(sms)))
    try:
        assert sms.value >= 8
        n = 30_000
        datas = [synth.generate(n, dim=2048, vocab=1000, n_stream_classes=100, seed=40 + j) for j in range(2)]
        torch.cuda.synchronize()
        prof = fx.make_default_profiles(1000)["cheap"]
        outs = [None, None]

        def run(j):
            fx.set_device(0)
            outs[j] = SP.device_ingest(datas[j], n, 4, 7.5, 100, 1000, prof)

        th = [threading.Thread(target=run, args=(j,)) for j in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for j in range(2):
            h = SP.host_stream(datas[j], n)
            ref = SP.oracle_ingest(h, 4, 7.5, 100, 1000, threads=os.cpu_count())
            rep = SP.compare(outs[j], ref, 1000)
            assert rep["mismatches"] == 0, rep["mismatch_by_field"]
    finally:
        _lib.check(L.fx_device_set_partitions(0, 0, None))
