"""Top SASS instructions by warp-stall samples with their dominant stall reasons.
usage: python tools/ncu_sass_hot.py REPORT [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h, d = rows[hi], rows[hi + 1:]
c = h.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[c]) for r in d)
print(rows[0][:2], "samples", tot)
for r in sorted(d, key=lambda r: -num(r[c]))[:top]:
    rs = sorted(((num(r[i]), h[i][6:]) for i in reasons), reverse=True)[:2]
    print(f"{num(r[c]):6d} {100 * num(r[c]) / max(tot, 1):5.1f}% {r[0][-5:]} {r[1][:60]:60s} {rs}")
