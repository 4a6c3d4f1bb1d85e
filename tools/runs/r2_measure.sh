#!/bin/bash
# Round-2 measurement batch (run on the GPU box from the repo root).
set -u
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/r2_bench_cfg3.json 2> $O/r2_bench_cfg3.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/r2_ref_cfg3.json 2> $O/r2_ref_cfg3.err
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/r2_bench_cfg2.json 2> $O/r2_bench_cfg2.err
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/r2_bench_cfg4.json 2> $O/r2_bench_cfg4.err
python bench.py --config 5 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > $O/r2_bench_cfg5_n4096.json 2> $O/r2_bench_cfg5.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches_cfg3.csv \
    python tools/prof_step.py 3 2 > $O/r2_launches_cfg3.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"conv_ws|conv_stack|conv_pad|ns_flow|tcg_tma|power_fused|emit_kernel|scale_bf16|conv_stem|pad_kernel" \
    -c 48 -o $O/r2_full_cfg3 python tools/prof_step.py 3 1 > $O/r2_full_cfg3.log 2>&1
python tools/ncu_summary.py $O/r2_full_cfg3.ncu-rep --json $O/r2_full_cfg3.json > $O/r2_full_cfg3.txt 2>&1
ncu -i $O/r2_full_cfg3.ncu-rep --page details --csv > $O/r2_full_cfg3_details.csv 2>/dev/null
gzip -f $O/r2_full_cfg3_details.csv
rm -f $O/r2_full_cfg3.ncu-rep     # gpurun copies back at most 64 MiB: keep the summaries
timeout 900 python tools/bench_rows.py > $O/r2_rows.jsonl 2> $O/r2_rows.err
echo done
