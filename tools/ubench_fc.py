"""Time the K1b kernels alone (CUPTI trace) on 65536 x 1000 x 2048 resident inputs."""
import collections, ctypes, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch
from torch.profiler import ProfilerActivity, profile
from paper_1801_03493_b200 import _lib
L = _lib.load()
n, V, D, K = 65536, 1000, 2048, 4
F = torch.randn(n, D, device="cuda"); W = torch.randn(V, D, device="cuda") / 45.0; b = torch.zeros(V, device="cuda")
tk = torch.empty(n, K, dtype=torch.int32, device="cuda"); cf = torch.empty(n, K, device="cuda"); fl = torch.empty(n, dtype=torch.uint8, device="cuda")
cs = torch.cuda.current_stream()
def call():
    _lib.check(L.fx_fc_topk_device(0, _lib.vp(cs.cuda_stream), n, D, V, K, _lib.vp(F.data_ptr()), _lib.vp(W.data_ptr()),
                                   _lib.vp(b.data_ptr()), _lib.vp(tk.data_ptr()), _lib.vp(cf.data_ptr()), _lib.vp(fl.data_ptr())))
call(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(3): call()
    torch.cuda.synchronize()
agg = collections.defaultdict(list)
for e in p.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "k_fc" in e.name:
        agg[e.name.split("(")[0]].append(e.device_time_total)
print(os.environ.get("FOCUS_B200_FCDBG", "0"), {k: round(sum(v) / len(v), 1) for k, v in agg.items()})
