"""Per-kernel device time of one C2 stream ingest + finalize, traced with
CUPTI through torch.profiler (real pipelined run, not ncu-serialised).
GPU box only:  python tools/trace_kernels.py [n_objects [T [M]]]  (C3 shape: 300000 5.0 100000)
Under programmatic dependent launch a kernel's traced duration includes the time its
CTAs wait for the previous grid: set FOCUS_B200_NOPDL=1 for per-kernel attribution."""
import collections
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1801_03493_b200 as fx
from paper_1801_03493_b200 import _lib, synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
T = float(sys.argv[2]) if len(sys.argv) > 2 else 7.5
M = int(sys.argv[3]) if len(sys.argv) > 3 else 100
data = synth.generate(n, dim=2048, vocab=1000, n_stream_classes=100, seed=0)
torch.cuda.synchronize()
prof = fx.make_default_profiles(1000)["cheap"]


def run():
    s = fx.ingest.Stream(2048, 16, 1000, 4, T, M, 0.01, _lib.FX_F32, 0, 0)
    s.set_rank_model(prof, 0)
    s.ingest_device(n, data.oids.data_ptr(), data.fids.data_ptr(), data.sigs.data_ptr(), data.feats.data_ptr(),
                    data.true_class.data_ptr())
    s.finalize()
    torch.cuda.synchronize()


run()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    run()
agg = collections.defaultdict(lambda: [0, 0.0])
tmin, tmax = None, None
for e in p.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"total kernel/memcpy time {tot / 1e3:.2f} ms")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k[:60]:60s} {v[0]:6d} {v[1] / 1e3:9.3f} ms  avg {v[1] / v[0]:8.2f} us")

# idle gaps between consecutive device activities (the engine runs on one stream)
ev = sorted([(e.time_range.start, e.time_range.end, e.name.split("(")[0].replace("void ", ""))
             for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda x: x[0])
gaps = collections.defaultdict(lambda: [0, 0.0])
span = ev[-1][1] - ev[0][0] if ev else 0
for a, b in zip(ev, ev[1:]):
    g = b[0] - a[1]
    if g > 0:
        key = f"{a[2][:28]} -> {b[2][:28]}"
        gaps[key][0] += 1
        gaps[key][1] += g
tg = sum(v[1] for v in gaps.values())
print(f"\ndevice span {span / 1e3:.2f} ms, idle gaps {tg / 1e3:.2f} ms")
for k, v in sorted(gaps.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{k:62s} {v[0]:6d} {v[1] / 1e3:8.3f} ms  avg {v[1] / v[0]:7.2f} us")

# timeline of three steady-state batches (k_snap_pack starts each batch)
marks = [i for i, e in enumerate(ev) if "k_snap_pack" in e[2]]
if len(marks) > 8:
    b0 = (3 * len(marks)) // 4  # steady state
    for bi in (b0, b0 + 1, b0 + 2):
        i0, i1 = marks[bi], marks[bi + 1]
        t0 = ev[i0][0]
        print(f"\nbatch {bi}: {(ev[i1][0] - t0) / 1e3 * 1e3:.1f} us")
        for a, b, nm in ev[i0:i1]:
            print(f"   {nm[:44]:44s} start {(a - t0):8.1f} us  end {(b - t0):8.1f} us  dur {(b - a):7.1f} us")
