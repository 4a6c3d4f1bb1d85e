"""Top CUDA source lines by warp-stall samples (all files) from an ncu report.
usage: python tools/ncu_src_hot.py REPORT [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname, hdr = [], None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if "Line No" in r or "# Line" in r or (r and r[0] == "#"):
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        try:
            c = hdr.index("Warp Stall Sampling (All Samples)")
            res.append((int(r[c] or 0), fname, r[0], r[1].strip()[:90]))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in res)
print("samples", tot)
for v, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{v:7d} {100 * v / max(tot, 1):5.1f}% {f}:{ln} {src}")
