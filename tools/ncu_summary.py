"""Per-launch summary of an ncu --set full report: duration, DRAM bytes
(read + write), L2 sectors, L2 / DRAM / tensor-pipe utilisation.
usage: python tools/ncu_summary.py REPORT [--json OUT]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "": 1, "%": 1}


def get(d, k):
    if k not in hdr:
        return float("nan")
    try:
        return float(d[k].replace(",", "")) * SCALE.get(units[hdr.index(k)], 1)
    except ValueError:
        return float("nan")


recs = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "").replace("orth::(anonymous namespace)::", "").replace("void ", "")
    name = name.split("(")[0] if "<" not in name.split("(")[0] else name.split("(")[0]
    recs.append(dict(
        kernel=name[:48], us=get(d, "gpu__time_duration.sum"),
        dram_bytes=get(d, "dram__bytes_read.sum") + get(d, "dram__bytes_write.sum"),
        l2_bytes=get(d, "lts__t_sectors.sum") * 32,
        l2_pct=get(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        dram_pct=get(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        tensor_pct=get(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        grid=get(d, "launch__grid_size")))
print(f"{'kernel':48s} {'us':>8s} {'DRAM MB':>9s} {'L2 MB':>9s} {'L2%':>6s} {'DRAM%':>6s} {'tensor%':>8s} {'grid':>5s}")
for r in recs:
    print(f"{r['kernel']:48s} {r['us']:8.1f} {r['dram_bytes'] / 1e6:9.2f} {r['l2_bytes'] / 1e6:9.2f} "
          f"{r['l2_pct']:6.1f} {r['dram_pct']:6.1f} {r['tensor_pct']:8.1f} {r['grid']:5.0f}")
if "--json" in sys.argv:
    json.dump(recs, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
