"""Aggregate warp-stall samples per CUDA source line from one or more
`ncu -i X --page source --csv --print-source cuda,sass` exports."""
import collections
import csv
import sys

agg = collections.defaultdict(float)
srcline = {}
tot = 0.0
for path in sys.argv[1:]:
    cur_file, hdr, last = None, None, None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) <= si:
            continue
        try:
            v = float(r[si].replace(",", "") or 0)
        except ValueError:
            continue
        if r[0]:
            last = (cur_file, int(r[0]))
            srcline[last] = r[1]
        agg[last] += v
        tot += v
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:45]:
    print(f"{v / tot:6.3f} {k[0]}:{k[1]:5d} {srcline.get(k, '').strip()[:110]}")
