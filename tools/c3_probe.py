"""C3-shaped stream (small T: every object seeds, M large) throughput probe."""
import os, sys, time
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch
import paper_1801_03493_b200 as fx
from paper_1801_03493_b200 import _lib, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
t = float(sys.argv[3]) if len(sys.argv) > 3 else 5.0
d = synth.generate(n, dim=2048, vocab=1000, n_stream_classes=100, seed=1)
torch.cuda.synchronize()
prof = fx.make_default_profiles(1000)["cheap"]
for rep in range(2):
    s = fx.ingest.Stream(2048, 16, 1000, 4, t, m, 0.01, _lib.FX_F32, 0, 0)
    if rep == 1:
        s.set_timing(True)
    s.set_rank_model(prof, 0)
    t0 = time.perf_counter()
    s.ingest_device(n, d.oids.data_ptr(), d.fids.data_ptr(), d.sigs.data_ptr(), d.feats.data_ptr(), d.true_class.data_ptr())
    ix, r = s.finalize()
    dt = time.perf_counter() - t0
    c = s.counters()
    print(f"n={n} m={m} t={t}: {n / dt:.0f} obj/s ({dt:.2f} s) clusters={r.clusters_emitted} live={c['nlive']} "
          f"exact={r.exact_rechecks} seq={c['seq_steps']} windows={c['windows']}", flush=True)
    if rep == 1:
        tm = s.timings()
        print({k: round(v, 1) for k, v in tm.items() if v}, flush=True)
        print({k: v for k, v in c.items() if k.startswith("cyc") or k in ("windows", "seq_steps", "nevict_total")}, flush=True)
