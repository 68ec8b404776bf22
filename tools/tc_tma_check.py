"""TC screen: TMA tiled staging vs cp.async staging -- outputs must be bit-identical
(same operands, same K order into TMEM).  GPU box: python tools/tc_tma_check.py"""
import ctypes, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
from paper_1801_03493_b200 import _lib
L = _lib.load()
L.fx_debug_screen_tc.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p]
rng = np.random.default_rng(0)
ok = True
for na, nb, D in [(1000, 300, 2048), (4096, 101, 2048), (130, 7, 200), (77, 129, 64), (20000, 1000, 256), (6000, 800, 2048)]:
    A = rng.standard_normal((na, D)).astype(np.float32)
    B = rng.standard_normal((nb, D)).astype(np.float32)
    outs = {}
    for mode in ("cp", "tma"):
        os.environ["FOCUS_B200_TCLOAD"] = mode
        out = np.zeros((na, nb), np.float32)
        rc = L.fx_debug_screen_tc(0, na, nb, D, A.ctypes.data, B.ctypes.data, out.ctypes.data)
        assert rc == 0, rc
        outs[mode] = out
    ref = (A.astype(np.float64) ** 2).sum(1)[:, None] + (B.astype(np.float64) ** 2).sum(1)[None] - 2 * A.astype(np.float64) @ B.T.astype(np.float64)
    same = all(np.array_equal(outs["cp"].view(np.uint32), outs[m].view(np.uint32)) for m in ("tma",))
    err = np.abs(outs["tma"] - ref).max() / np.abs(ref).max()
    print(f"na={na} nb={nb} D={D}: bit-identical={same} max rel err vs fp64={err:.2e}")
    ok &= same and err < 1e-2
print("OK" if ok else "MISMATCH")
