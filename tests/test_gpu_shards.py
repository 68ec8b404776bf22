"""Stream-sharded queries over DEVICE sessions.

* NCCL, world 1: ShardedQuery's NCCL branch (query_device / fetch_device +
  two all_gathers of CUDA tensors) on real device sessions; the merged result
  must equal each session's own query and the CPU oracle.
* gloo, world 2 on one GPU (FOCUS_B200_ONE_GPU-style: both ranks drive
  cuda:0; NCCL refuses two ranks on one device): every rank ingests its own
  streams on the device, answers for them, and the merge equals the
  single-process oracle results in stream order.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

N_STREAMS = 3
QUERIES = [(0, 1), (3, 4), (7, 2), (11, None)]


def _stream_inputs(si):
    from oracle import oracle as O
    from oracle import streamgen
    spec = streamgen.Spec(n_objects=1500, dim=32, vocab=30, n_stream_classes=12, seed=60 + si)
    st = streamgen.generate(spec)
    prof = O.default_profiles(30)["cheap"]
    dup = O.dup_flags(st.fids, st.sigs, 0.01)
    keep = ~dup
    feats = np.zeros((st.oids.size, 32), np.float32)
    feats[keep] = O.extract_features(prof, si, st.oids[keep], st.feats[keep]).astype(np.float32)
    return st, feats, dup


def _oracle(si, cls, kx):
    from oracle import oracle as O
    st, feats, dup = _stream_inputs(si)
    prof = O.default_profiles(30)["cheap"]
    keep = ~dup
    topk = np.zeros((st.oids.size, 4), np.int32)
    topk[keep] = O.classify_topk(prof, si, st.oids[keep], st.true_class[keep], 4)
    res = O.ingest(st.oids, st.fids, st.sigs, feats, topk, 4, 0.9, 25, is_dup=dup)
    gt = {int(o): int(c) for o, c in zip(st.oids, st.true_class)}
    q = O.OracleSession(res.clusters, 4, 30, gt).execute_query(cls, kx)
    return (si, list(q["frame_ids"]), list(q["object_ids"]), q["gt_inferences"], q["clusters_examined"],
            q["clusters_matched"])


def _device_session(si):
    import paper_1801_03493_b200 as fx
    st, feats, _ = _stream_inputs(si)
    cfg = fx.Config("cheap", k=4, l_s=30, t=0.9, m=25)
    idx, _, _ = fx.ingest_arrays(st.oids, st.fids, st.sigs, feats, cfg, fx.make_default_profiles(30)["cheap"],
                                 vocab=30, seed=si, true_class=st.true_class.astype(np.int32))
    objs = {int(o): fx.DetectedObject(int(o), int(f), 0.0, np.zeros(1), np.zeros(1), int(c))
            for o, f, c in zip(st.oids, st.fids, st.true_class)}
    return fx.QuerySession(idx, fx.make_default_profiles(30)["gt"], objs)


def _rows(merged):
    return [(r.stream_index, r.frame_ids.tolist(), r.object_ids.tolist(), r.gt_inferences, r.clusters_examined,
             r.clusters_matched) for r in merged]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_nccl_world1_device_sessions():
    import paper_1801_03493_b200 as fx
    from paper_1801_03493_b200 import shards
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sess = {si: _device_session(si) for si in range(N_STREAMS)}
        sq = shards.ShardedQuery(sess, N_STREAMS)
        for cls, kx in QUERIES:
            got = _rows(sq.query(fx.QueryRequest(cls, k_x=kx)))
            assert got == [_oracle(si, cls, kx) for si in range(N_STREAMS)]
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1801_03493_b200 as fx
        from paper_1801_03493_b200 import shards
        fx.set_device(0)
        sess = {si: _device_session(si) for si in shards.local_streams(N_STREAMS, rank, world)}
        sq = shards.ShardedQuery(sess, N_STREAMS)
        queue.put((rank, [_rows(sq.query(fx.QueryRequest(c, k_x=k))) for c, k in QUERIES]))
    except Exception as e:  # surface the failure in the parent
        queue.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(400)
def test_gloo_world2_device_sessions_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=360) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert not isinstance(got[r], str), got[r]
    for qi, (cls, kx) in enumerate(QUERIES):
        exp = [_oracle(si, cls, kx) for si in range(N_STREAMS)]
        assert got[0][qi] == exp
        assert got[1][qi] == exp
