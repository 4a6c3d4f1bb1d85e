"""Build profiles/r1_traffic.json (the `traffic` field of bench.py's roofline) from an
ncu --set full summary of one cfg2 construction + forward chain (tools/ncu_summary.py --json).
usage: python tools/make_traffic.py SUMMARY.json SOURCE_NOTE > profiles/r1_traffic.json"""
import json
import sys

sys.path.insert(0, ".")
from synth import configs  # noqa: E402

recs = json.load(open(sys.argv[1]))
note = sys.argv[2] if len(sys.argv) > 2 else ""
conv = [r for r in recs if r["kernel"].split("::")[-1].startswith("conv_")]
orth = [r for r in recs if any(k in r["kernel"] for k in ("power_fused", "scale_bf16", "ns_flow", "ns_persist"))]
out = {configs.NAMES[2]: {
    "conv apply": {"dram_bytes_per_launch": sum(r["dram_bytes"] for r in conv) / max(1, len(conv)),
                   "l2_bytes_per_launch": sum(r["l2_bytes"] for r in conv) / max(1, len(conv)),
                   "launches": len(conv)},
    "orth_orthogonalize (power + NS)": {"dram_bytes_per_launch": sum(r["dram_bytes"] for r in orth), "launches": 1},
    "source": note}}
print(json.dumps(out, indent=1))
