"""Per-kernel mean durations from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

agg, hdr = defaultdict(list), None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg[d["Kernel Name"].split("(")[0][-48:]].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:48s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:9.1f} us  share={sum(v) / tot:6.1%}")
