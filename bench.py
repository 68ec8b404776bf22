"""Benchmark: Focus ingest hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = ingest of one whole synthetic stream through K0 (pixel diff) +
K1a (rank-model top-K) + K2 (screen / resolve / fold) + seal + K3 (index
build): the C2 workload (1 stream x 1M objects, D=2048, V=1000, K=4, T=7.5,
M=100) per GPU.  Multi-GPU: one process per GPU, each owns its own stream
(natural stream sharding, no data-path collective) -> weak scaling; value =
objects of all ranks / max-over-ranks device time.

`value` times fx_ingest_device + fx_finalize with inputs resident in HBM
(CUDA events on the library's stream).  `e2e` times the host-buffer C-ABI
call (fx_ingest from pinned host memory, H2D inside, index read back).
`cpu_baseline` runs the CPU oracle port (oracle/) on a bounded prefix of the
same workload; `--impl reference` times that port as the reference arm.
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD = dict(n=1_000_000, dim=2048, vocab=1000, n_stream_classes=100, k=4, t=7.5, m=100)
METRIC = "ingest objects/sec (top-K+cluster+index)"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.path = os.path.join(REPO, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        try:
            rows = [l.strip().split(",") for l in open(self.path) if l.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_sample(n_sample: int, seed: int, threads: int, h: dict | None = None):
    """Time the CPU oracle port (reference algorithm restated in C + numpy) on
    the first n_sample objects of the workload (`h`: the GPU arm's own stream
    copied to the host; else the same generator on the CPU).  Returns objects/s."""
    from oracle import oracle as O
    if h is None:
        from paper_1801_03493_b200 import synth
        st = synth.generate(n_sample, dim=WORKLOAD["dim"], vocab=WORKLOAD["vocab"],
                            n_stream_classes=WORKLOAD["n_stream_classes"], seed=seed, device="cpu")
        h = dict(oids=st.oids.numpy(), fids=st.fids.numpy(), sigs=st.sigs.numpy(), feats=st.feats.numpy(),
                 true_class=st.true_class.numpy())
    oids, fids = h["oids"][:n_sample], h["fids"][:n_sample]
    sigs, feats, tcls = h["sigs"][:n_sample], h["feats"][:n_sample], h["true_class"][:n_sample]
    prof = O.default_profiles(WORKLOAD["vocab"])["cheap"]
    O.set_threads(threads)
    k = WORKLOAD["k"]
    t0 = time.perf_counter()
    dup = O.dup_flags(fids, sigs, 0.01)
    keep = ~dup
    topk = np.zeros((oids.size, k), np.int32)
    topk[keep] = O.classify_topk(prof, 0, oids[keep], tcls[keep], k)
    res = O.ingest(oids, fids, sigs, feats, topk, k, WORKLOAD["t"], WORKLOAD["m"], is_dup=dup, with_centroids=False)
    O.build_postings(res.clusters)
    dt = time.perf_counter() - t0
    return n_sample / dt, dt, len(res.clusters)


def _focusidx():
    """The unmodified reference package from baseline/_ref (pip-installed
    there once; it travels with the repo snapshot), or None."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "focusidx")) and ref not in sys.path:
        sys.path.append(ref)
    try:
        import focusidx  # noqa: F401
        from focusidx import classifiers, clustering, core, index, ingest, query, streamio
        return dict(classifiers=classifiers, clustering=clustering, core=core, index=index, ingest=ingest,
                    query=query, streamio=streamio)
    except Exception:
        return None


def reference_python_ingest(h: dict, n: int):
    """The reference's own ingest_stream (focusidx, unmodified, 1 core) on the
    first n objects of the host stream: the rank-model cheap profile with
    feature noise 0 (the rows already are the cheap CNN's output, as on the
    device), seed 0.  Returns (objects/s, seconds, clusters) or None."""
    R = _focusidx()
    if R is None:
        return None
    from dataclasses import replace
    V = WORKLOAD["vocab"]
    profs = R["classifiers"].make_default_profiles(V)
    profs["cheap"] = replace(profs["cheap"], feature_noise_sigma=0.0)
    DO = R["core"].DetectedObject
    objs = [DO(int(h["oids"][i]), int(h["fids"][i]), 0.0, h["sigs"][i], h["feats"][i], int(h["true_class"][i]))
            for i in range(n)]
    cfg = R["core"].Config("cheap", k=WORKLOAD["k"], l_s=V, t=WORKLOAD["t"], m=WORKLOAD["m"])
    hdr = R["streamio"].StreamHeader("cam0", 30.0, WORKLOAD["dim"], h["sigs"].shape[1], V)
    t0 = time.perf_counter()
    idx, rep = R["ingest"].ingest_stream(hdr, objs, cfg, profs, 0.01, 0)
    dt = time.perf_counter() - t0
    return n / dt, dt, rep.clusters_emitted


def parity_and_c5(data, W, local, args):
    """Rank 0, after the timed region: (1) the bench's own stream ingested on
    the device at K = 4 vs the CPU oracle, bit for bit (oracle/scale_parity.py);
    (2) C5 (BASELINE configs[4]): the same stream ingested at K = 8, every
    class x k_x in {1,2,4,8} queried with a FRESH QuerySession, each result
    compared with the oracle session; (3) the CPU query latency beside it (the
    oracle port and, when baseline/_ref holds it, the reference's own
    QuerySession)."""
    import paper_1801_03493_b200 as fx
    from oracle import oracle as O
    from oracle import scale_parity as SP
    n, V, t, m = W["n"], W["vocab"], W["t"], W["m"]
    prof = fx.make_default_profiles(V)["cheap"]
    t0 = time.perf_counter()
    dev4 = SP.device_ingest(data, n, W["k"], t, m, V, prof, device=local)
    h = SP.host_stream(data, n)
    t1 = time.perf_counter()
    ref8 = SP.oracle_ingest(h, 8, t, m, V, threads=os.cpu_count())
    t2 = time.perf_counter()
    par = SP.compare(dev4, SP.derive_k(ref8, W["k"]), V)
    del dev4
    par.update(oracle_s=round(t2 - t1, 2), oracle_threads=os.cpu_count(),
               note="the timed workload's stream (all objects), device K=4 ingest vs the CPU oracle run at K=8 "
                    "(K=4 expectations derived: top-K prefix, class ranks <= 4; clustering is K-independent)")
    # C5: K = 8 index, fresh session per query, parity per query
    s8 = fx.ingest.Stream(W["dim"], 16, V, 8, t, m, 0.01, fx._lib.FX_F32, local, 0)
    s8.set_rank_model(prof, 0)
    s8.ingest_device(n, data.oids.data_ptr(), data.fids.data_ptr(), data.sigs.data_ptr(), data.feats.data_ptr(),
                     data.true_class.data_ptr())
    dix8, _ = s8.finalize()
    cfg8 = fx.Config("cheap", k=8, l_s=V, t=t, m=m)
    tix = fx.TopKIndex(fx.IndexHeader("cam0", W["dim"], V, n, cfg8), device=dix8)
    labels = h["true_class"].astype(np.int32)
    gt = fx.make_default_profiles(V)["gt"]
    osess = O.OracleSession(ref8.clusters, 8, V, dict(zip(h["oids"].tolist(), labels.tolist())))
    classes = list(range(V)) if args.queries < 0 else list(range(min(V, args.queries)))
    lat, bad, nq, frames = [], 0, 0, []
    for kx in (1, 2, 4, 8):
        for c in classes:
            q0 = time.perf_counter()
            sess = fx.QuerySession(tix, gt, None, labels=labels)
            fr, ob, st = sess.query_arrays(fx.QueryRequest(c, k_x=kx))
            lat.append((time.perf_counter() - q0) * 1e3)
            del sess
            osess.cache = {}
            exp = osess.execute_query(c, kx)
            nq += 1
            frames.append(fr.size)
            if (not np.array_equal(fr, np.asarray(exp["frame_ids"], np.int64))
                    or not np.array_equal(ob, np.asarray(exp["object_ids"], np.int64))
                    or st != (exp["gt_inferences"], exp["clusters_examined"], exp["clusters_matched"])):
                bad += 1
    lat = np.array(lat)
    c5 = {"queries": nq, "k_x": [1, 2, 4, 8], "index_k": 8, "classes": len(classes),
          "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
          "mean_ms": float(lat.mean()), "max_frames": int(max(frames)), "mean_frames": float(np.mean(frames)),
          "parity": {"queries_checked": nq, "mismatches": bad},
          "timing": "host wall clock per query: fresh QuerySession (labels gathered on the device) + lookup + "
                    "verify + expansion + ids copied to host"}
    # CPU query latency beside it (fresh session per query)
    cpu_q = {}
    sub = classes if len(classes) <= 200 else list(range(0, V, max(1, V // 200)))
    ql = []
    for kx in (1, 2, 4, 8):
        for c in sub:
            q0 = time.perf_counter()
            osess.cache = {}
            osess.execute_query(c, kx)
            ql.append((time.perf_counter() - q0) * 1e3)
    cpu_q["oracle_port"] = {"p50_ms": float(np.percentile(ql, 50)), "p99_ms": float(np.percentile(ql, 99)),
                            "mean_ms": float(np.mean(ql)), "queries": len(ql), "cores": 1}
    R = _focusidx()
    if R is not None:
        Cl = R["clustering"].Cluster
        rcl = [Cl(cluster_id=c.cluster_id, centroid=np.zeros(1), member_object_ids=list(c.member_object_ids),
                  frame_ids=list(c.frame_ids), class_best_rank=dict(c.class_best_rank),
                  centroid_member_id=c.centroid_member_id, sealed=True) for c in ref8.clusters]
        ridx = R["index"].build(rcl, R["index"].IndexHeader("cam0", W["dim"], V, n, R["core"].Config(
            "cheap", k=8, l_s=V, t=t, m=m)))
        DO = R["core"].DetectedObject
        objs = {c.centroid_member_id: DO(c.centroid_member_id, 0, 0.0, np.zeros(1), np.zeros(1),
                                         int(labels[c.centroid_member_id])) for c in ref8.clusters}
        rgt = R["classifiers"].make_default_profiles(V)["gt"]
        ql = []
        for kx in (1, 2, 4, 8):
            for c in sub:
                q0 = time.perf_counter()
                R["query"].QuerySession(ridx, rgt, objs).execute_query(R["query"].QueryRequest(c, k_x=kx))
                ql.append((time.perf_counter() - q0) * 1e3)
        cpu_q["reference_python"] = {"p50_ms": float(np.percentile(ql, 50)), "p99_ms": float(np.percentile(ql, 99)),
                                     "mean_ms": float(np.mean(ql)), "queries": len(ql), "cores": 1,
                                     "what": "focusidx.query.QuerySession (unmodified, baseline/_ref) over the "
                                             "same K=8 index, fresh session per query"}
    c5["cpu_baseline"] = cpu_q
    del tix, dix8, s8
    return par, c5, h


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_sample = args.ref_sample
    from paper_1801_03493_b200 import synth
    st = synth.generate(n_sample, dim=WORKLOAD["dim"], vocab=WORKLOAD["vocab"],
                        n_stream_classes=WORKLOAD["n_stream_classes"], seed=0, device="cpu")
    h = dict(oids=st.oids.numpy(), fids=st.fids.numpy(), sigs=st.sigs.numpy(), feats=st.feats.numpy(),
             true_class=st.true_class.numpy())
    for _ in range(args.warmup):
        cpu_sample(n_sample, 0, threads, h)
    vals = []
    for _ in range(args.steps):
        v, dt, ncl = cpu_sample(n_sample, 0, threads, h)
        vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "objects/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": n_sample / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 prefix: first {n_sample} objects of 1 stream (D=2048, V=1000, K=4, T=7.5, "
                               f"M=100); the reference algorithm as the C/OpenMP oracle port (oracle/), "
                               f"{threads} host threads on the per-insert distance row -- a stronger baseline "
                               f"than the single-threaded reference Python", **WORKLOAD},
        "cpu_baseline": {"value": value, "unit": "objects/s", "cores": threads, "kind": "port",
                         "sample": f"first {n_sample} objects of the C2 stream per step, {threads} threads"},
        "e2e": {"value": value, "unit": "objects/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--objects", dest="n", type=int, default=WORKLOAD["n"], help="objects per stream")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample", type=int, default=200000,
                    help="objects of the single-core oracle-port cpu_baseline (BASELINE.md §2: 200k prefix)")
    ap.add_argument("--ref-python-sample", type=int, default=10000,
                    help="objects of the unmodified reference Python ingest timed beside it (0 = skip)")
    ap.add_argument("--ref-sample", type=int, default=50000)
    ap.add_argument("--no-check", action="store_true", help="skip the parity + C5 legs (oracle on the host)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--queries", type=int, default=-1, help="classes queried (x3 k_x values); -1 = every class, 0 = skip")
    ap.add_argument("--backend", default="nccl", help="process-group backend for N > 1 (nccl; gloo for checks)")
    ap.add_argument("--no-fc", action="store_true", help="skip the K1b FC head sub-benchmark")
    ap.add_argument("--multi-streams", type=int, default=8, help="concurrent engines for the C4-shape line (<=1: skip)")
    ap.add_argument("--multi-objects", type=int, default=1_000_000, help="objects per engine in the C4-shape line")
    ap.add_argument("--multi-partitions", type=int, default=4,
                    help="SM partitions (green contexts) = engines ingesting concurrently in the C4-shape line")
    ap.add_argument("--c3-objects", type=int, default=300_000,
                    help="objects of the C3-shape line (T=5, M=100k: every object seeds; 0 = skip)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1801_03493_b200 as fx
    from paper_1801_03493_b200 import _lib, synth

    ws, rank, local = _dist()
    if os.environ.get("FOCUS_B200_ONE_GPU"):  # multi-rank logic check on a 1-GPU box (with --backend gloo)
        local = 0
    torch.cuda.set_device(local)
    fx.set_device(local)
    if ws > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.backend)
    W = dict(WORKLOAD, n=args.n)
    data = synth.generate(W["n"], dim=W["dim"], vocab=W["vocab"], n_stream_classes=W["n_stream_classes"], seed=rank)
    torch.cuda.synchronize()
    cfg = fx.Config("cheap", k=W["k"], l_s=W["vocab"], t=W["t"], m=W["m"])
    prof = fx.make_default_profiles(W["vocab"])["cheap"]
    L = _lib.load()

    def make_stream():
        s = fx.ingest.Stream(W["dim"], 16, W["vocab"], W["k"], W["t"], W["m"], 0.01, _lib.FX_F32, local, args.batch)
        s.set_rank_model(prof, 0)
        return s

    host_split = {"ingest_call_ms": 0.0, "finalize_call_ms": 0.0}

    def step(s):
        t0 = time.perf_counter()
        s.ingest_device(W["n"], data.oids.data_ptr(), data.fids.data_ptr(), data.sigs.data_ptr(),
                        data.feats.data_ptr(), data.true_class.data_ptr())
        t1 = time.perf_counter()
        out = s.finalize()
        t2 = time.perf_counter()
        host_split["ingest_call_ms"] += (t1 - t0) * 1e3
        host_split["finalize_call_ms"] += (t2 - t1) * 1e3
        if os.environ.get("BENCH_DEBUG"):
            print(f"step: ingest {(t1 - t0) * 1e3:.1f} ms finalize {(t2 - t1) * 1e3:.1f} ms "
                  + " ".join(f"{k}={v:.1f}" for k, v in s.timings().items() if k.startswith("host")),
                  file=sys.stderr, flush=True)
        return out

    # warm-up
    for _ in range(args.warmup):
        s = make_stream()
        step(s)
        del s
    # one step = create the stream engine, ingest the whole stream, finalize
    # (seal + index build); the engine and its index are released right after
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    host_split.update(ingest_call_ms=0.0, finalize_call_ms=0.0)
    launches0 = L.fx_kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    reports = []
    last = last_idx = None
    with Clocks(local) as clk:
        ev0.record()
        for i in range(args.steps):
            s = make_stream()
            idx, rep_i = step(s)
            reports.append(rep_i)
            if i == args.steps - 1:
                last, last_idx = s, idx
            del s, idx
        ev1.record()
        torch.cuda.synchronize()
    launches = L.fx_kernel_launches() - launches0
    host_split = {k: v / args.steps for k, v in host_split.items()}
    t_ms = ev0.elapsed_time(ev1)
    dev_red = "cuda" if args.backend == "nccl" else "cpu"
    if ws > 1:
        tt = torch.tensor([t_ms], device=dev_red)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.barrier()
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    value = W["n"] * ws * args.steps / (t_ms / 1e3)
    rep = reports[-1]
    # per-phase breakdown from one extra, instrumented run of the same step
    # (the timed steps run without the phase events, which sit between kernels)
    inst = make_stream()
    inst.set_timing(True)
    step(inst)
    phases = inst.timings()
    counters = inst.counters()
    del inst

    # roofline: algorithmic bytes per launch / average launch
    # duration from the library's CUDA events on its own stream.  The headline
    # kernel is the K2 TF32 screen (the clustering kernel the north star names;
    # it streams every classified feature once from HBM); the other kernels
    # are listed with theirs.  The dominant phase by time is the resolve, a
    # single-CTA latency-bound pass with no meaningful byte roofline.
    D, n_cls = W["dim"], rep.objects_classified
    nb = max(1.0, phases["batches"])
    peak, peak_kind = _peaks()
    feat_bytes = 4.0 * D * n_cls
    kern = {  # phase -> (algorithmic bytes per step, what)
        "screen": (feat_bytes + 4.0 * counters["dc"], "k_screen_tc: features streamed once + distance row written"),
        "screen_summary": (feat_bytes, "k_rowpass: each feature row re-read once (refine + residual columns)"),
        "fold": (feat_bytes + 8.0 * D * phases["batches"] * 100, "k_fold: member rows into the float64 sums"),
        "seal": (feat_bytes, "k_seal_dist: every featured member vs its final centroid"),
        "k0_k1a": (128.0 * rep.objects_seen + (12.0 + 4 * W["k"]) * n_cls, "K0 pixel diff + K1a rank top-K"),
        "index": (12.0 * W["k"] * n_cls, "K3 class sets + postings"),
    }
    rl = {}
    for k, (byts, what) in kern.items():
        ms = phases.get(k, 0.0)
        if ms > 0:
            ach = byts / (ms / 1e3) / 1e9
            rl[k] = {"what": what, "ms_per_step": ms, "achieved_gbs": ach, "frac": ach / peak}
    scr_ms = phases["screen"]
    scr_ach = kern["screen"][0] / (scr_ms / 1e3) / 1e9
    traffic = None
    try:  # dram bytes per launch of the same kernel from the committed ncu --set full capture
        tj = json.load(open(os.path.join(REPO, "profiles", "ncu_traffic.json")))
        traffic = float(next(v for k, v in tj.items() if "k_screen_tc" in k))
    except Exception:
        pass
    roofline = {"kernel": "k_screen_tc (K2 TF32 distance screen)", "bound": "hbm", "achieved": scr_ach, "peak": peak,
                "unit": "GB/s", "frac": scr_ach / peak, "traffic": traffic,
                "traffic_note": "dram read+write bytes per launch, ncu --set full of a steady-state batch "
                                "(profiles/r02f_ncu_full_metrics.txt, B = 8192 classified objects: algorithmic "
                                "4*D*8192 + 4*8192*101 = 70.4 MB, so ~1.26x): the TMA boxes also stage the "
                                "duplicate objects' rows between the batch's classified rows", "peak_kind": peak_kind,
                "launches_per_step": int(nb), "bytes_per_launch": kern["screen"][0] / nb,
                "avg_launch_us": scr_ms * 1e3 / nb,
                "per_kernel": rl,
                "phase_ms_per_step": {k: v for k, v in phases.items() if k != "batches" and not k.startswith("host")},
                "dominant_phase": max(("screen", "screen_resid", "screen_summary", "resolve", "fold", "seal"),
                                      key=lambda k: phases.get(k, 0.0)),
                "host_wall_ms_per_step": host_split}

    # end-to-end through the host-buffer C ABI
    e2e = None
    if args.e2e_steps > 0:
        ho = data.oids.cpu().pin_memory()
        hf = data.fids.cpu().pin_memory()
        hs = data.sigs.cpu().pin_memory()
        ht = data.true_class.cpu().pin_memory()
        # the cheap CNN runs after pixel differencing: its feature output holds
        # the classified objects' rows only (FX_FEATS_COMPACT); the generator's
        # intended duplicates must be exactly what K0 finds
        k0 = fx.ingest.dup_flags(hf.numpy(), hs.numpy(), 0.01)
        assert np.array_equal(k0, data.is_dup.cpu().numpy()), "generator duplicates != K0 duplicates"
        hx = data.feats[~data.is_dup].cpu().pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in (ho, hf, hs, hx, ht))
        e_times = []
        d2h = 0
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s = fx.ingest.Stream(W["dim"], 16, W["vocab"], W["k"], W["t"], W["m"], 0.01, _lib.FX_F32, local,
                                 args.batch)
            s.set_rank_model(prof, 0)
            s.ingest(ho.numpy(), hf.numpy(), hs.numpy(), hx.numpy(), true_class=ht.numpy(), compact=True)
            dix, r = s.finalize()
            ex = dix.export(centroids=True)
            d2h = sum(a.nbytes for a in ex.values())
            t1 = time.perf_counter()
            if i > 0:
                e_times.append(t1 - t0)
            del s, dix
        et = float(np.mean(e_times))
        if ws > 1:
            tt = torch.tensor([et], device=dev_red)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            et = float(tt.item())
        e2e_v = W["n"] * ws / et
        e2e = {"value": e2e_v, "unit": "objects/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "timing": "host wall clock around fx_ingest(host ptrs, FX_FEATS_COMPACT: the classified objects' "
                         "feature rows, as the cheap CNN emits them; H2D chunked and overlapped with the ingest) "
                         "+ fx_finalize + index export, pinned inputs, max over ranks"}

    # C5-style query latency on the ingested index: lookup(k_x) -> GT verify ->
    # member expansion, fresh session per query; over N ranks every query is
    # answered for all N streams and merged with the NCCL all-gathers
    # (paper_1801_03493_b200/shards.py).  Host wall clock per query, ids on host.
    qres = None
    if args.queries != 0:
        from paper_1801_03493_b200 import shards
        header = fx.IndexHeader(stream_id=f"cam{rank}", dim=W["dim"], vocab=W["vocab"], n_objects=W["n"], config=cfg)
        tix = fx.TopKIndex(header, device=last_idx)
        sess = fx.QuerySession(tix, fx.make_default_profiles(W["vocab"])["gt"], None,
                               labels=data.true_class.cpu().numpy())
        classes = np.arange(W["vocab"], dtype=np.int64)  # C5: every class x k_x
        if 0 < args.queries < W["vocab"]:
            classes = np.random.default_rng(123).choice(classes, size=args.queries, replace=False)
        sq = shards.ShardedQuery({rank: sess}, ws) if ws > 1 else None
        lat, nfr = [], []
        for kx in (1, 2, 4):
            for c in classes.tolist():
                req = fx.QueryRequest(int(c), k_x=kx)
                if ws > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                if sq is not None:
                    res = sq.query(req)
                    nf = sum(r.frame_ids.size for r in res)
                else:
                    sess.reset()
                    fr, ob, st = sess.query_arrays(req)
                    nf = fr.size
                lat.append((time.perf_counter() - t0) * 1e3)
                nfr.append(nf)
        lat = np.array(lat)
        if ws > 1:
            lt = torch.tensor(lat, device="cuda" if args.backend == "nccl" else "cpu")
            dist.all_reduce(lt, op=dist.ReduceOp.MAX)
            lat = lt.cpu().numpy()
        qres = {"queries": int(lat.size), "k_x": [1, 2, 4], "p50_ms": float(np.percentile(lat, 50)),
                "p99_ms": float(np.percentile(lat, 99)), "mean_ms": float(lat.mean()),
                "mean_frames": float(np.mean(nfr)), "max_frames": int(np.max(nfr)),
                "merge": f"{args.backend} all_gather x2 over {ws} ranks" if ws > 1 else "single stream",
                "timing": "host wall clock per query (fresh session, ids copied to host), max over ranks"}
        del sess, tix
    del last, last_idx  # the last timed step's engine and index

    # Engines still referenced by earlier legs' objects (indexes, sessions in
    # reference cycles) count as live on the device, and an engine that is not
    # alone drops programmatic dependent launch (run_batches: multi_inline):
    # free them before each leg so its number does not depend on GC timing.
    gc.collect()

    # C4 shape on this GPU: several stream engines ingesting concurrently
    # ("the 1/2/4-GPU points of C4 run 8/4/2 engines per GPU"),
    # one host thread per engine, each on its own CUDA stream; the streams are
    # the device-generated stream of this rank with distinct seeds.
    msres = None
    if args.multi_streams > 1:
        from concurrent.futures import ThreadPoolExecutor
        nms = args.multi_streams
        nobj = min(W["n"], args.multi_objects)
        datas = [synth.generate(nobj, dim=W["dim"], vocab=W["vocab"], n_stream_classes=W["n_stream_classes"],
                                seed=1000 + rank * nms + j) for j in range(nms)]
        torch.cuda.synchronize()

        # SM partitions (CUDA green contexts, fx_device_set_partitions): worker w
        # runs engines w, w + P, ... in partition w, so concurrent engines never
        # share SMs.  Without them, concurrent engines starve each other's
        # large-shared-memory CTAs (the single-CTA resolve, the TC screen) for
        # up to seconds at a time.
        nparts = max(1, min(nms, args.multi_partitions))
        sms = ctypes.c_int32(0)
        if nparts > 1:
            _lib.check(_lib.load().fx_device_set_partitions(local, nparts, ctypes.byref(sms)))

        def one(j, part):
            fx.set_device(local)
            d = datas[j]
            sj = fx.ingest.Stream(W["dim"], 16, W["vocab"], W["k"], W["t"], W["m"], 0.01, _lib.FX_F32, local,
                                  args.batch, partition=part)
            sj.set_rank_model(prof, 0)
            sj.ingest_device(nobj, d.oids.data_ptr(), d.fids.data_ptr(), d.sigs.data_ptr(), d.feats.data_ptr(),
                             d.true_class.data_ptr())
            ix, rp = sj.finalize()
            del ix, sj
            return rp.objects_seen

        def worker(w):
            return sum(one(j, w + 1 if nparts > 1 else 0) for j in range(w, nms, nparts))

        with ThreadPoolExecutor(max_workers=nparts) as pool:
            list(pool.map(worker, range(nparts)))  # warm-up
            dts = []
            for _ in range(3):  # median of 3 wall-clock runs (host thread scheduling jitter)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                seen = sum(pool.map(worker, range(nparts)))
                torch.cuda.synchronize()
                dts.append(time.perf_counter() - t0)
            dt = sorted(dts)[1]
        if nparts > 1:
            _lib.check(_lib.load().fx_device_set_partitions(local, 0, None))
        if ws > 1:
            tt = torch.tensor([dt], device=dev_red)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        msres = {"streams_per_gpu": nms, "sm_partitions": nparts, "sms_per_partition": int(sms.value) or 148,
                 "objects_per_stream": nobj, "objects_per_s": seen * ws / dt, "wall_s": dt, "all_runs_s": dts,
                 "note": "C4 shape: engines per GPU, one host thread per SM partition (CUDA green context) running "
                         "its engines one after another, inputs resident, wall clock (median of 3 runs), max over "
                         "ranks"}
        del datas

    gc.collect()  # see above: no leftover engine may turn the C3 engine's PDL off
    # C3 shape (BASELINE configs[2]: M = 100 k, T = 5 -- every object seeds,
    # the live set saturates at 100 k and every batch evicts) on a bounded
    # prefix, inputs resident; parity of this path: tests/test_gpu_seeds.py
    c3res = None
    if args.c3_objects > 0:
        n3 = args.c3_objects
        d3 = synth.generate(n3, dim=W["dim"], vocab=W["vocab"], n_stream_classes=W["n_stream_classes"],
                            seed=1 + rank)
        torch.cuda.synchronize()
        t3 = []
        for _ in range(2):  # the first run pays the allocations of the 100 k-slot engine
            s3 = fx.ingest.Stream(W["dim"], 16, W["vocab"], W["k"], 5.0, 100_000, 0.01, _lib.FX_F32, local, 0)
            s3.set_rank_model(prof, 0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s3.ingest_device(n3, d3.oids.data_ptr(), d3.fids.data_ptr(), d3.sigs.data_ptr(), d3.feats.data_ptr(),
                             d3.true_class.data_ptr())
            ix3, rp3 = s3.finalize()
            torch.cuda.synchronize()
            t3.append(time.perf_counter() - t0)
            c3c = s3.counters()
            del ix3, s3
        dt3 = min(t3)
        if ws > 1:
            tt = torch.tensor([dt3], device=dev_red)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt3 = float(tt.item())
        c3res = {"objects_per_stream": n3, "objects_per_s": n3 * ws / dt3, "wall_s": dt3,
                 "clusters": rp3.clusters_emitted, "evictions": int(c3c["nevict_total"]),
                 "distance_computations": rp3.distance_computations,
                 "note": "C3 shape: T=5.0, M=100000 (every object seeds, live set saturated), "
                         "wall clock incl. engine create/finalize, inputs resident, best of 2"}
        del d3

    # K1b FC classifier head (north star kernel 1) on resident features:
    # logits over V classes, top-K; tensor-pipe roofline against TF32 dense
    fcres = None
    if not args.no_fc:
        nfc = min(1 << 18, W["n"])
        Fd = data.feats[:nfc]
        gfc = torch.Generator(device="cuda")
        gfc.manual_seed(7)
        Wt = torch.randn(W["vocab"], W["dim"], device="cuda", generator=gfc) / float(np.sqrt(W["dim"]))
        bt = 0.1 * torch.randn(W["vocab"], device="cuda", generator=gfc)
        tk = torch.empty(nfc, W["k"], dtype=torch.int32, device="cuda")
        cf = torch.empty(nfc, W["k"], dtype=torch.float32, device="cuda")
        fl = torch.empty(nfc, dtype=torch.uint8, device="cuda")
        cs = torch.cuda.current_stream()

        def fc_call():
            _lib.check(L.fx_fc_topk_device(local, _lib.vp(cs.cuda_stream), nfc, W["dim"], W["vocab"], W["k"],
                                           _lib.vp(Fd.data_ptr()), _lib.vp(Wt.data_ptr()), _lib.vp(bt.data_ptr()),
                                           _lib.vp(tk.data_ptr()), _lib.vp(cf.data_ptr()), _lib.vp(fl.data_ptr())))
        fc_call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record(cs)
        for _ in range(reps):
            fc_call()
        e1.record(cs)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        flops = 2.0 * W["vocab"] * W["dim"] * nfc
        tf = flops / (ms / 1e3) / 1e12
        try:
            bf16 = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["bf16_tflops"])
            tf32_peak, pk = bf16 / 2.0, "MEASURED_PEAKS bf16 dense / 2 (TF32 is half the BF16 rate)"
        except Exception:
            tf32_peak, pk = 1125.0, "fallback: nominal 2.25 PF bf16 / 2"
        # per-kernel split of one more call (CUPTI): the logits kernel's own tensor-pipe fraction
        per_k = {}
        try:
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                fc_call()
                torch.cuda.synchronize()
            for ev in prof.events():
                if ev.device_type == torch.autograd.DeviceType.CUDA and "k_fc" in ev.name:
                    nm = ev.name.split("(")[0].replace("void ", "").replace("fx::", "")
                    per_k[nm] = per_k.get(nm, 0.0) + ev.device_time_total / 1e3
        except Exception as e:  # profiler unavailable: the split is optional
            per_k = {"unavailable": str(e)[:80]}
        fc_kernels = {k: {"ms": v, "tflops": flops / (v / 1e3) / 1e12 if "tcp" in k or "fc_tc" in k else None,
                          "frac": (flops / (v / 1e3) / 1e12) / tf32_peak if "tcp" in k or "fc_tc" in k else None}
                      for k, v in per_k.items() if isinstance(v, float)}
        fcres = {"objects": nfc, "vocab": W["vocab"], "dim": W["dim"], "k": W["k"], "ms": ms, "kernels": fc_kernels,
                 "objects_per_s": nfc / (ms / 1e3), "achieved_tflops": tf, "peak_tflops": tf32_peak,
                 "frac": tf / tf32_peak, "peak_kind": pk, "flagged": int(fl.sum().item()),
                 "bound": "tensor", "note": "TF32 tcgen05 logits + float64 re-score of the candidates"}

    # feature noise (extract_feature, classifiers.py:152-158) on the device:
    # 65 k objects x D normals, float32 features in, float64 out; one numpy
    # object timed beside it (the reference's per-object call)
    noiseres = None
    if not args.no_fc:
        nn_ = min(1 << 16, W["n"])
        Fn = data.feats[:nn_]
        On = data.oids[:nn_]
        outn = torch.empty(nn_, W["dim"], dtype=torch.float64, device="cuda")
        flg = torch.zeros(1, dtype=torch.int64, device="cuda")
        csn = torch.cuda.current_stream()

        def noise_call():
            _lib.check(L.fx_extract_features_device(local, nn_, W["dim"], _lib.vp(On.data_ptr()), _lib.vp(Fn.data_ptr()),
                                                    _lib.FX_F32, W["dim"], 0.05, 0, _lib.vp(outn.data_ptr()),
                                                    W["dim"], _lib.vp(flg.data_ptr()), _lib.vp(csn.cuda_stream)))
        noise_call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(csn)
        for _ in range(3):
            noise_call()
        e1.record(csn)
        torch.cuda.synchronize()
        msn = e0.elapsed_time(e1) / 3
        fh = Fn[:200].cpu().numpy()
        oh = On[:200].cpu().numpy()
        q0 = time.perf_counter()
        for i in range(200):
            fh[i].astype(np.float64) + 0.05 * np.random.default_rng([0, int(oh[i]), 1]).standard_normal(W["dim"])
        cpu_s = (time.perf_counter() - q0) / 200
        noiseres = {"objects": nn_, "dim": W["dim"], "ms": msn, "objects_per_s": nn_ / (msn / 1e3),
                    "normals_per_s": nn_ * W["dim"] / (msn / 1e3),
                    "hbm_gbs": nn_ * W["dim"] * (4 + 8) / (msn / 1e3) / 1e9, "flagged": int(flg.item()),
                    "cpu_numpy_objects_per_s": 1.0 / cpu_s,
                    "note": "fx_extract_features_device: SeedSequence + PCG64 + ziggurat (bit-exact numpy), "
                            "f32 features in, f64 out; cpu = numpy default_rng(...).standard_normal per object, 1 core"}
        del outn

    parity = c5 = h = None
    if rank == 0 and not args.no_check:
        parity, c5, h = parity_and_c5(data, W, local, args)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        nsamp = min(args.cpu_sample, W["n"])
        v, dt, ncl = cpu_sample(nsamp, 0, 1, h)
        cpu = {"value": v, "unit": "objects/s", "cores": 1, "kind": "port",
               "sample": f"first {nsamp} objects of the timed C2 stream ({dt:.1f} s, single thread: the C "
                         f"oracle port, 1 core per stream as BASELINE.md §2 states)"}
        if args.ref_python_sample > 0:
            if h is None:
                from oracle import scale_parity as SP
                h = SP.host_stream(data, min(W["n"], args.ref_python_sample))
            rp = reference_python_ingest(h, min(args.ref_python_sample, h["oids"].size))
            if rp is not None:
                cpu["reference_python"] = {
                    "value": rp[0], "unit": "objects/s", "cores": 1, "clusters": rp[2],
                    "sample": f"first {min(args.ref_python_sample, h['oids'].size)} objects of the same stream "
                              f"({rp[1]:.1f} s): focusidx.ingest.ingest_stream, unmodified (baseline/_ref)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "objects/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic (device generator, reference model)",
            "config": {"workload": "C2: 1 stream x 1M objects per GPU, D=2048, V=1000, K=4, T=7.5, M=100",
                       "streams_per_gpu": 1, "parallelism": f"stream-sharded x{ws}",
                       "l2": "inputs (8 GB features/stream) exceed L2; no flush", **W},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
            "query": qres, "c5_query_sweep": c5, "parity": parity, "k1b_fc_head": fcres, "feature_noise": noiseres, "multi_stream": msres,
            "c3_shape": c3res,
            "gpu_launches": int(launches),
            "ingest": {"clusters": rep.clusters_emitted, "classified": rep.objects_classified,
                       "distance_computations": rep.distance_computations, "exact_rechecks": rep.exact_rechecks,
                       "fast_decisions": counters["fast"],
                       "resolve_profile": {k: counters[k] for k in counters if k.startswith(("cyc_", "conf_"))
                                           or k in ("windows", "seq_steps", "fast_batches") or k.startswith("fold_")}},
        }
        print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
