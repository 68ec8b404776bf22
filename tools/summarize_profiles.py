"""Turn a round's ncu captures (gpurun_out/) into the committed summaries
under profiles/:  python tools/summarize_profiles.py r01"""
import csv
import io
import json
import os
import subprocess
import sys

T = sys.argv[1] if len(sys.argv) > 1 else "r01"
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(REPO, "gpurun_out"), os.path.join(REPO, "profiles")
os.makedirs(P, exist_ok=True)
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for w in WANT:
            for i, name in enumerate(h):
                if name == w or (w.startswith("sm__pipe_tensor") and name.startswith("sm__pipe_tensor") and "pct" in name):
                    d[name] = r[i] + (" " + units[i] if units[i] else "")
        res.append(d)
    return res


traffic = {}
lines = []
for rep in (f"full_{T}.ncu-rep", f"fc_{T}.ncu-rep"):
    path = os.path.join(G, rep)
    if not os.path.exists(path):
        continue
    lines.append(f"## {rep}")
    for d in raw(path):
        lines.append(json.dumps(d))
        def nbytes(v):
            num, unit = (v.split() + ["byte"])[:2]
            return float(num.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        try:
            traffic.setdefault(d["kernel"], []).append(nbytes(d["dram__bytes_read.sum"]) +
                                                      nbytes(d["dram__bytes_write.sum"]))
        except (KeyError, ValueError, IndexError):
            pass
open(os.path.join(P, f"{T}_ncu_full_metrics.txt"), "w").write("\n".join(lines) + "\n")
json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
lc = os.path.join(G, f"launches_{T}.csv")
if os.path.exists(lc):
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_launch_summary.py"), lc], capture_output=True,
                         text=True).stdout
    open(os.path.join(P, f"{T}_launches_n200k.txt"), "w").write(out)
print("wrote", os.listdir(P))
