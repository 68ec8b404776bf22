"""Diagnostic: host vs device time of one C2 stream ingest, with and without
an nvidia-smi sampler running alongside (GPU box only)."""
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch

import paper_1801_03493_b200 as fx
from paper_1801_03493_b200 import _lib, synth

n = int(os.environ.get("N", "1000000"))
W = dict(dim=2048, vocab=1000, k=4, t=7.5, m=100)
data = synth.generate(n, dim=2048, vocab=1000, n_stream_classes=100, seed=0)
torch.cuda.synchronize()
prof = fx.make_default_profiles(1000)["cheap"]


def one(tag):
    s = fx.ingest.Stream(2048, 16, 1000, 4, 7.5, 100, 0.01, _lib.FX_F32, 0, int(os.environ.get("BATCH", "0")))
    s.set_rank_model(prof, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.ingest_device(n, data.oids.data_ptr(), data.fids.data_ptr(), data.sigs.data_ptr(), data.feats.data_ptr(),
                    data.true_class.data_ptr())
    t1 = time.perf_counter()
    s.finalize()
    t2 = time.perf_counter()
    ph = s.timings()
    print(f"{tag}: ingest {1e3*(t1-t0):.1f} ms finalize {1e3*(t2-t1):.1f} ms | " +
          " ".join(f"{k}={v:.1f}" for k, v in ph.items() if k != "_"), flush=True)


for i in range(int(os.environ.get("REPS", "3"))):
    one(f"plain{i}")
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                     stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
for i in range(int(os.environ.get("REPS", "3"))):
    one(f"smi{i}")
p.terminate()
p.wait()
for i in range(2):
    one(f"plain_after{i}")
