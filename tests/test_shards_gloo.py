"""Stream-sharded query merge with world_size 2 over gloo on
CPU: per-stream results computed on their owner ranks and all-gathered must
equal the single-process results in stream order.  The per-stream results
here come from the CPU oracle (the device sessions produce the same arrays;
the GPU path all-gathers them over NCCL with the same packing)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from oracle import streamgen

N_STREAMS = 5


def _stream_results(si: int, cls: int, kx: int):
    spec = streamgen.Spec(n_objects=700, dim=16, vocab=30, n_stream_classes=10, seed=40 + si)
    st = streamgen.generate(spec)
    prof = O.default_profiles(30)["cheap"]
    dup = O.dup_flags(st.fids, st.sigs, 0.01)
    keep = ~dup
    feats = np.zeros((st.oids.size, 16))
    feats[keep] = O.extract_features(prof, 0, st.oids[keep], st.feats[keep])
    topk = np.zeros((st.oids.size, 4), np.int32)
    topk[keep] = O.classify_topk(prof, 0, st.oids[keep], st.true_class[keep], 4)
    res = O.ingest(st.oids, st.fids, st.sigs, feats, topk, 4, 0.6, 20, is_dup=dup)
    gt = {int(o): int(c) for o, c in zip(st.oids, st.true_class)}
    q = O.OracleSession(res.clusters, 4, 30, gt).execute_query(cls, kx)
    return (si, np.asarray(q["frame_ids"], np.int64), np.asarray(q["object_ids"], np.int64),
            (q["gt_inferences"], q["clusters_examined"], q["clusters_matched"]))


def _worker(rank, world, port, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1801_03493_b200 import shards
        out = []
        for cls, kx in [(0, 1), (3, 4), (7, 2)]:
            parts = [_stream_results(si, cls, kx) for si in shards.local_streams(N_STREAMS, rank, world)]
            merged = shards.merge(parts, N_STREAMS)
            out.append([(r.stream_index, r.frame_ids.tolist(), r.object_ids.tolist(), r.gt_inferences,
                         r.clusters_examined, r.clusters_matched) for r in merged])
        queue.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_owner_assignment():
    from paper_1801_03493_b200 import shards
    assert shards.local_streams(5, 0, 2) == [0, 2, 4] and shards.local_streams(5, 1, 2) == [1, 3]
    assert sorted(sum((shards.local_streams(8, r, 3) for r in range(3)), [])) == list(range(8))


@pytest.mark.timeout(300)
def test_gloo_world2_merge_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for qi, (cls, kx) in enumerate([(0, 1), (3, 4), (7, 2)]):
        exp = []
        for si in range(N_STREAMS):
            _, fr, ob, st = _stream_results(si, cls, kx)
            exp.append((si, fr.tolist(), ob.tolist(), *st))
        assert got[0][qi] == exp
        assert got[1][qi] == exp
