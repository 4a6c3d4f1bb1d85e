"""Top SASS lines by warp-stall samples from an ncu report (one launch).
usage: python tools/ncu_hot.py REPORT [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r)
hdr = rows[hdr_i]
data = rows[hdr_i + 1:]
col = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
vals = [(int(r[col]) if r[col].isdigit() else 0, r) for r in data if len(r) > col]
tot = sum(v for v, _ in vals)
print(rows[0][:2], "total samples", tot)
for v, r in sorted(vals, key=lambda x: -x[0])[:top]:
    print(f"{v:6d} {100.0 * v / max(tot, 1):5.1f}%  {r[0][-5:]}  {r[src][:90]}")
