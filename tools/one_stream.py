"""Ingest one device-generated C2-shaped stream (for sanitizer runs).
    python tools/one_stream.py [n] [seed] [T] [M] [engines]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_03493_b200 as fx  # noqa: E402
from paper_1801_03493_b200 import _lib, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1004
T = float(sys.argv[3]) if len(sys.argv) > 3 else 7.5
M = int(sys.argv[4]) if len(sys.argv) > 4 else 100
E = int(sys.argv[5]) if len(sys.argv) > 5 else 1
datas = [synth.generate(n, seed=seed + j) for j in range(E)]
torch.cuda.synchronize()
prof = fx.make_default_profiles(1000)["cheap"]


def one(j):
    d = datas[j]
    s = fx.ingest.Stream(2048, 16, 1000, 4, T, M, 0.01, _lib.FX_F32, 0, 0)
    s.set_rank_model(prof, 0)
    s.ingest_device(n, d.oids.data_ptr(), d.fids.data_ptr(), d.sigs.data_ptr(), d.feats.data_ptr(),
                    d.true_class.data_ptr())
    ix, rp = s.finalize()
    c = s.counters()
    cl, _, _ = s.object_results(n, 4)
    return rp.clusters_emitted, c["exact"], c["windows"], int(np.bitwise_xor.reduce(cl.astype(np.int64) * 2654435761))


t0 = time.time()
if E == 1:
    print(one(0))
else:
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(E) as p:
        print(list(p.map(one, range(E))))
print("elapsed", time.time() - t0)
