"""Timeline of one C2 ingest step (CUPTI via torch.profiler): per-kernel device
time and the idle gaps between consecutive device activities, attributed to
the activity that precedes each gap.  Diagnostic only."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03493_b200 as fx  # noqa: E402
from paper_1801_03493_b200 import _lib, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
data = synth.generate(n, dim=2048, vocab=1000, n_stream_classes=100, seed=0)
prof = fx.make_default_profiles(1000)["cheap"]


def run():
    s = fx.ingest.Stream(2048, 16, 1000, 4, 7.5, 100, 0.01, _lib.FX_F32, 0, 0)
    s.set_rank_model(prof, 0)
    s.ingest_device(n, data.oids.data_ptr(), data.fids.data_ptr(), data.sigs.data_ptr(), data.feats.data_ptr(),
                    data.true_class.data_ptr())
    return s.finalize()


run()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as p:
    run()
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
p.export_chrome_trace("gpurun_out/trace_ingest.json")
ev = json.load(open("gpurun_out/trace_ingest.json"))["traceEvents"]
dev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
dev.sort(key=lambda e: e["ts"])
busy = collections.defaultdict(float)
gaps = collections.defaultdict(float)
cnt = collections.Counter()
for i, e in enumerate(dev):
    name = e["name"].split("(")[0].split("<")[0][:60]
    busy[name] += e["dur"]
    cnt[name] += 1
    if i + 1 < len(dev):
        g = dev[i + 1]["ts"] - (e["ts"] + e["dur"])
        if g > 0:
            gaps[name] += g
span = dev[-1]["ts"] + dev[-1]["dur"] - dev[0]["ts"]
print(f"span {span / 1e3:.1f} ms, busy {sum(busy.values()) / 1e3:.1f} ms, gaps {sum(gaps.values()) / 1e3:.1f} ms")
print("busy by activity (ms):")
for k, v in sorted(busy.items(), key=lambda x: -x[1])[:18]:
    print(f"  {k:60s} {cnt[k]:6d} {v / 1e3:9.2f}")
print("idle gap after activity (ms):")
for k, v in sorted(gaps.items(), key=lambda x: -x[1])[:15]:
    print(f"  {k:60s} {v / 1e3:9.2f}")
