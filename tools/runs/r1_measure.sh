#!/bin/bash
# Round-1 measurement batch (run on the GPU box from the repo root).
set -u
O=gpurun_out
python -m pytest tests -m gpu -q -x > $O/r1_pytest_gpu.log 2>&1
tail -2 $O/r1_pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $O/r1_bench_cfg2.json 2> $O/r1_bench_cfg2.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/r1_ref_cfg2.json 2> $O/r1_ref_cfg2.err
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $O/r1_bench_cfg3.json 2>/dev/null
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/r1_bench_cfg4.json 2>/dev/null
python bench.py --config 5 --n 2048 --steps 5 --warmup 3 --no-cpu-baseline > $O/r1_bench_cfg5_n2048.json 2>/dev/null
python bench.py --config 5 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > $O/r1_bench_cfg5_n4096.json 2>/dev/null
ORTH_NO_PDL=1 python tools/kprof.py 2 5 > $O/r1_kprof_cfg2.txt 2>&1
ORTH_NO_PDL=1 python tools/kprof.py 3 3 > $O/r1_kprof_cfg3.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r1_launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"conv_|ns_persist|ns_flow|tcg_tma|power_fused|emit|cvt_|scale_" -c 30 \
    -o $O/r1_full_cfg2 python tools/prof_conv.py 1 > /dev/null 2>&1
echo done
