"""Concurrent stream engines on one GPU (the C4 shape): wall clock for
N = 1, 2, 4, 8 engines, each on its own host thread and CUDA stream.

    python tools/multi_probe.py [--objects 1000000] [--streams 1,2,4,8]
"""
import argparse
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1801_03493_b200 as fx  # noqa: E402
from paper_1801_03493_b200 import _lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--objects", type=int, default=1_000_000)
    ap.add_argument("--streams", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--serial", action="store_true", help="one host thread runs the engines one after another")
    ap.add_argument("--verify", action="store_true", help="compare every run's results with the first (solo) run")
    ap.add_argument("--counters", action="store_true", help="print each engine's resolve/fold counters")
    ap.add_argument("--trace", type=int, default=0, help="CUPTI-trace this many extra runs at the largest N")
    ap.add_argument("--trace-stall", type=int, default=0,
                    help="trace up to this many runs at the largest N; report the longest device activities of a "
                         "run slower than 1 s")
    ap.add_argument("--partitions", type=int, default=0, help="SM partitions (green contexts) for the engines")
    a = ap.parse_args()
    ns = [int(x) for x in a.streams.split(",")]
    nmax = max(ns)
    datas = [synth.generate(a.objects, seed=1000 + j) for j in range(nmax)]
    torch.cuda.synchronize()
    prof = fx.make_default_profiles(1000)["cheap"]
    if a.partitions > 1:
        import ctypes
        sms = ctypes.c_int32(0)
        _lib.check(_lib.load().fx_device_set_partitions(0, a.partitions, ctypes.byref(sms)))
        print(f"{a.partitions} SM partitions of {sms.value} SMs", flush=True)

    solo = {}

    def one(j):
        fx.set_device(0)
        d = datas[j]
        t0 = time.perf_counter()
        s = fx.ingest.Stream(2048, 16, 1000, 4, 7.5, 100, 0.01, _lib.FX_F32, 0, 0)
        s.set_rank_model(prof, 0)
        t1 = time.perf_counter()
        s.ingest_device(a.objects, d.oids.data_ptr(), d.fids.data_ptr(), d.sigs.data_ptr(), d.feats.data_ptr(),
                        d.true_class.data_ptr())
        t2 = time.perf_counter()
        ix, rp = s.finalize()
        t3 = time.perf_counter()
        if a.verify:
            import numpy as np
            cl, _, _ = s.object_results(a.objects, 4)
            ex = ix.export(centroids=True)
            h = hash((cl.tobytes(), ex["centroids"].tobytes(), ex["reps"].tobytes()))
            if j in solo and solo[j] != h:
                print(f"  MISMATCH engine {j}: concurrent result differs from its solo run", flush=True)
            solo.setdefault(j, h)
        if a.counters:
            c = s.counters()
            print(f"  engine {j}: " + " ".join(f"{k}={c[k]}" for k in (
                "windows", "seq_steps", "exact", "fast", "cyc_passA", "cyc_passB", "cyc_passCD", "cyc_passE",
                "cyc_seq", "fold_wait_cyc", "fold_chain_cyc", "fold_slot_cyc", "fold_rows")), flush=True)
        tm = s.timings()
        del ix, s
        t4 = time.perf_counter()
        if t2 - t1 > 1.0:  # a stalled ingest: where did the host wait?
            print(f"  SLOW engine {j}: ingest {(t2 - t1)*1e3:.0f} ms; host phases (ms): " +
                  " ".join(f"{k}={v:.1f}" for k, v in tm.items() if k.startswith("host") and v > 1.0), flush=True)
        return (t1 - t0, t2 - t1, t3 - t2, t4 - t3)

    with ThreadPoolExecutor(max_workers=nmax) as pool:
        for j in range(nmax):  # solo reference runs (one engine at a time)
            one(j)
        for n in ns:
            for r in range(a.reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if a.serial:
                    parts = [one(j) for j in range(n)]
                else:
                    parts = list(pool.map(one, range(n)))
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                mx = [max(p[i] for p in parts) for i in range(4)]
                print(f"N={n} rep={r} wall={dt*1e3:.1f} ms  {n * a.objects / dt / 1e6:.2f} M obj/s  "
                      f"max create={mx[0]*1e3:.1f} ingest={mx[1]*1e3:.1f} finalize={mx[2]*1e3:.1f} "
                      f"destroy={mx[3]*1e3:.1f} ms", flush=True)
        for r in range(a.trace_stall):
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as p:
                t0 = time.perf_counter()
                list(pool.map(one, range(nmax)))
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
            print(f"STALLPROBE run {r}: wall {dt*1e3:.1f} ms", flush=True)
            if dt < 1.0:
                continue
            ev = sorted([(e.time_range.start, e.time_range.end, e.name.split("(")[0].replace("void ", "")[:60])
                         for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda x: x[0])
            t00 = ev[0][0]
            longest = sorted(ev, key=lambda x: x[0] - x[1])[:12]
            for s0, s1, nm in longest:
                print(f"   {nm:60s} start {(s0 - t00)/1e3:10.3f} ms dur {(s1 - s0)/1e3:10.3f} ms", flush=True)
            # idle stretches of the whole device
            busy_end, gaps = ev[0][1], []
            for s0, s1, nm in ev[1:]:
                if s0 > busy_end:
                    gaps.append((s0 - busy_end, busy_end - t00, nm))
                busy_end = max(busy_end, s1)
            for g, at, nm in sorted(gaps, reverse=True)[:8]:
                print(f"   device idle {g/1e3:10.3f} ms at {at/1e3:10.3f} ms (then {nm})", flush=True)
            break
        for r in range(a.trace):
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as p:
                t0 = time.perf_counter()
                list(pool.map(one, range(nmax)))
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
            ev = [e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA]
            tot = {}
            for e in ev:
                nm = e.name.split("(")[0].replace("void ", "")[:50]
                c, t, m = tot.get(nm, (0, 0.0, 0.0))
                d = e.device_time_total
                tot[nm] = (c + 1, t + d, max(m, d))
            print(f"TRACE run {r}: wall {dt*1e3:.1f} ms, {len(ev)} device events", flush=True)
            for nm, (c, t, m) in sorted(tot.items(), key=lambda x: -x[1][1])[:15]:
                print(f"   {nm:50s} n={c:6d} total={t/1e3:10.2f} ms  max={m/1e3:9.3f} ms", flush=True)


if __name__ == "__main__":
    main()
