"""Build profiles/r2_traffic.json (the `traffic` field of bench.py's roofline: DRAM bytes per launch of each
kernel group, keyed like bench.py's kernel groups) from an ncu --set full summary (tools/ncu_summary.py --json).
usage: python tools/make_traffic.py SUMMARY.json CONFIG SOURCE_NOTE > profiles/r2_traffic.json"""
import json
import sys

recs = json.load(open(sys.argv[1]))
cfg = sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
GROUPS = {"conv_ws<256": "conv_ws<256>", "conv_ws<128": "conv_ws<128>", "conv_pad<64, true": "conv_pad<64,swapped>", "conv_pad<64, 1, 0>": "conv_pad<64,swapped>",
          "conv_pad<64, 0, 1>": "conv_pad<64,row>", "conv_pad<64, false, true>": "conv_pad<64,row>", "tcg_flow": "compose",
          "conv_stack": "conv_stack (+pad_kernel)", "conv_stem": "conv_stem_tc", "ns_flow": "ns", "ns_persist": "ns",
          "power_fused": "power", "emit_kernel": "emit", "scale_bf16": "scale", "tcg_tma": "compose"}
out = {}
for key, name in GROUPS.items():
    rs = [r for r in recs if key in r["kernel"]]
    if rs:
        out[name] = {"dram_bytes_per_launch": sum(r["dram_bytes"] for r in rs) / len(rs),
                     "l2_bytes_per_launch": sum(r["l2_bytes"] for r in rs) / len(rs),
                     "tensor_pct": sum(r["tensor_pct"] for r in rs) / len(rs), "launches_captured": len(rs)}
out["source"] = note
print(json.dumps({f"config {cfg}": out}, indent=1))
