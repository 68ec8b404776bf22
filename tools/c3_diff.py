"""C3-shape stream: write cluster_of + counters of one ingest (mode from
FOCUS_B200_TCLOAD) to gpurun_out/c3_<tag>.npz for cross-mode comparison."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np, torch
import paper_1801_03493_b200 as fx
from paper_1801_03493_b200 import _lib, synth
n, m, t, tag = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), sys.argv[4]
d = synth.generate(n, dim=2048, vocab=1000, n_stream_classes=100, seed=1)
torch.cuda.synchronize()
s = fx.ingest.Stream(2048, 16, 1000, 4, t, m, 0.01, _lib.FX_F32, 0, 0)
s.set_rank_model(fx.make_default_profiles(1000)["cheap"], 0)
s.ingest_device(n, d.oids.data_ptr(), d.fids.data_ptr(), d.sigs.data_ptr(), d.feats.data_ptr(), d.true_class.data_ptr())
c = s.counters()
try:
    ix, r = s.finalize()
    ok = True
except Exception as e:
    print("finalize:", e)
    ok = False
cl, dup, tk = s.object_results(n, 4)
np.savez(f"gpurun_out/c3_{tag}.npz", cl=cl, err=np.array([0 if ok else 1]))
print(tag, {k: c[k] for k in ("nlive", "next_cid", "dc", "nevict_total", "exact", "err", "seq_steps")})
