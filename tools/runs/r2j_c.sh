#!/bin/bash
set -u
O=gpurun_out
ncu --set full --import-source on --clock-control none \
    -k regex:"conv_ws|conv_stack|conv_pad|ns_flow|tcg_flow|power_fused|emit_kernel|scale_bf16|conv_stem|pad_kernel" \
    -c 48 -o $O/r2j_full_cfg3 python tools/prof_step.py 3 1 > $O/r2j_full_cfg3.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py $O/r2j_full_cfg3.ncu-rep --json $O/r2j_full_cfg3.json > $O/r2j_full_cfg3.txt 2>&1
ncu -i $O/r2j_full_cfg3.ncu-rep --page details --csv > $O/r2j_full_cfg3_details.csv 2>/dev/null
gzip -f $O/r2j_full_cfg3_details.csv
rm -f $O/r2j_full_cfg3.ncu-rep
