"""Top warp-stall SASS lines from `ncu -i X --page source --csv --print-source sass` output."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h) and x[0] != "Address"]
si, ai, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
f = lambda v: float(v.replace(",", "") or 0)
tot = sum(f(x[si]) for x in rows)
print("total samples", tot)
for x in sorted(rows, key=lambda x: -f(x[si]))[:n]:
    print(f"{f(x[si]) / tot:6.3f} {x[ie]:>9s} {x[0]} {x[ai][:100]}")
