"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
iS, iA, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [(int(r[iA] or 0), r[hdr.index("Address")], r[iS].strip(), r[iE]) for r in rows[1:] if len(r) == len(hdr)]
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
for s, a, src, ex in sorted(data, reverse=True)[:top]:
    print(f"{s / tot:6.1%} {a[-5:]} {src[:70]:70s} exec={ex}")
