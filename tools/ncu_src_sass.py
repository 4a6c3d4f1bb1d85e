"""Attribute SASS warp-stall samples to CUDA source lines (ncu --print-source cuda,sass).
usage: python tools/ncu_src_sass.py REPORT [top] [launch_index]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 4 and r[0] == "Line No")
c = hdr.index("Warp Stall Sampling (All Samples)")
agg, cur, fname = collections.Counter(), None, ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) != len(hdr) or r[0] == "Line No":
        continue
    if r[0]:
        cur = f"{fname}:{r[0]}: {r[1].strip()[:80]}"
    elif r[2] and r[c].isdigit() and cur:
        agg[cur] += int(r[c])
tot = sum(agg.values())
for k, v in agg.most_common(top):
    print(f"{v:6d} {100 * v / max(1, tot):5.1f}%  {k}")
