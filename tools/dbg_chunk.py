import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, golden_util as GU, paper_1801_03493_b200 as fx
c = GU.load("small_d64"); st = c.stream
cfg = fx.Config("cheap", k=4, l_s=1000, t=1.0, m=20)
prof = fx.make_default_profiles(1000)["cheap"]
s = fx.ingest.Stream(64, 16, 1000, 4, 1.0, 20, 0.01, 0, None, 128)
s.set_rank_model(prof, 0)
cuts = [0, 7, 8, 500, 1001, 1002, 1999, 2000]
for a, b in zip(cuts, cuts[1:]):
    try:
        s.ingest(st.oids[a:b].copy(), st.fids[a:b].copy(), np.ascontiguousarray(st.sigs[a:b]), np.ascontiguousarray(c.feats[a:b]), true_class=st.true_class[a:b].astype(np.int32))
    except Exception as e:
        print("chunk", a, b, "failed:", repr(e), "dups:", c.g["is_dup"][a:b].sum()); raise
print("ok")
try:
    dix, rep = s.finalize()
    print("finalize ok", rep.clusters_emitted, rep.distance_computations)
except Exception as e:
    print("finalize failed:", repr(e))
