"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.

usage: python tools/ncu_launch_summary.py gpurun_out/launches.csv > profiles/<round>_launches.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
fx_tot = sum(v[1] for k, v in agg.items() if k.startswith("fx::"))
print(f"# {sys.argv[1]}: per-kernel gpu__time_duration.sum (ncu, serialised, --clock-control none)")
print(f"# total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches; fx:: kernels {fx_tot:.1f} us")
print(f"{'kernel':58s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:58]:58s} {v[0]:8d} {v[1]:11.1f} {v[1] / v[0]:9.2f} {v[1] / tot:6.3f}")
