"""K1b on the bench's own inputs (first 256 k objects of the C2 stream, W ~ N(0,1/D),
bias 0.1 N(0,1)); CUPTI per-kernel averages and the TF32 rate of the whole head."""
import collections, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
from paper_1801_03493_b200 import _lib, synth
L = _lib.load()
n, V, D, K = int(os.environ.get("N", 1 << 18)), 1000, 2048, 4
data = synth.generate(n, dim=D, vocab=V, n_stream_classes=100, seed=0)
F = data.feats[:n]
g = torch.Generator(device="cuda"); g.manual_seed(7)
W = torch.randn(V, D, device="cuda", generator=g) / float(np.sqrt(D)); b = 0.1 * torch.randn(V, device="cuda", generator=g)
tk = torch.empty(n, K, dtype=torch.int32, device="cuda"); cf = torch.empty(n, K, device="cuda"); fl = torch.empty(n, dtype=torch.uint8, device="cuda")
cs = torch.cuda.current_stream()
def call():
    _lib.check(L.fx_fc_topk_device(0, _lib.vp(cs.cuda_stream), n, D, V, K, _lib.vp(F.data_ptr()), _lib.vp(W.data_ptr()),
                                   _lib.vp(b.data_ptr()), _lib.vp(tk.data_ptr()), _lib.vp(cf.data_ptr()), _lib.vp(fl.data_ptr())))
call(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(cs)
for _ in range(3): call()
e1.record(cs); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(3): call()
    torch.cuda.synchronize()
agg = collections.defaultdict(list)
for e in p.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "k_fc" in e.name:
        agg[e.name.split("(")[0]].append(e.device_time_total)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FOCUS_B200_FC"))
print(tag, f"ms={ms:.3f} TFLOP/s={2.0*n*V*D/ms/1e9:.1f} flagged={int(fl.sum())}",
      {k: round(sum(v) / len(v), 1) for k, v in agg.items()}, flush=True)
