"""Debug: per-cluster centroid bit comparison for one golden case (GPU box)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np

import golden_util as GU
from oracle import oracle as O
import test_gpu_parity as T

name = sys.argv[1] if len(sys.argv) > 1 else "c3_shape_d2048"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 0
c = GU.load(name)
idx, rep, stream = T._run_case(c, batch=batch)
ex = idx.device.export()
h = GU.row_hash(ex["centroids"])
bad = np.nonzero(h != c.g["cl_centroid_h64"])[0]
print(name, "clusters", len(h), "bad", len(bad), "first", bad[:10].tolist())
st = c.stream
dup = c.g["is_dup"]
res = O.ingest(st.oids, st.fids, st.sigs, c.feats, np.asarray(c.g["topk"], np.int32), c.cfg["k"], c.cfg["t"],
               c.cfg["m"], is_dup=dup)
for i in bad[:5]:
    ref = res.clusters[i].centroid
    got = ex["centroids"][i]
    diff = np.nonzero(ref.view(np.uint64) != got.view(np.uint64))[0]
    mem = ex["mem_off"][i + 1] - ex["mem_off"][i]
    print(f"cluster {i}: members {mem} ndiff {len(diff)} dims {diff[:8].tolist()} ref {ref[diff[:3]]} got {got[diff[:3]]}")
