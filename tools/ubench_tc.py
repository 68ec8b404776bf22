"""Time k_screen_tc alone (CUPTI trace) on a 4096 x 101 x 2048 problem via fx_debug_screen_tc."""
import ctypes, os, sys, collections
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_1801_03493_b200 import _lib
L = _lib.load()
L.fx_debug_screen_tc.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
na, nb, D = 4096, 101, 2048
A = np.random.randn(na, D).astype(np.float32); B = np.random.randn(nb, D).astype(np.float32); out = np.zeros((na, nb), np.float32)
torch.cuda.init()
for _ in range(2): L.fx_debug_screen_tc(0, na, nb, D, A.ctypes.data, B.ctypes.data, out.ctypes.data)
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(5): L.fx_debug_screen_tc(0, na, nb, D, A.ctypes.data, B.ctypes.data, out.ctypes.data)
ts = [e.device_time_total for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA and "k_screen_tc" in e.name]
print(os.environ.get("FOCUS_B200_TCDBG", "0"), os.environ.get("FOCUS_B200_TCSPLIT", "auto"), "k_screen_tc us:", [round(t, 1) for t in ts])
