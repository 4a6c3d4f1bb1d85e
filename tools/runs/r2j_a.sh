#!/bin/bash
# Round-2 final measurement, part A (GPU tests, benches, rows); parts B and C run ncu (one ncu per call).
set -u
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/r2j_pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -3 $O/r2j_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2j_smoke.txt 2>&1; echo "smoke rc=$?"
python bench.py > $O/r2j_bench_default.json 2> $O/r2j_bench_default.err; echo "bench rc=$?"
python bench.py --steps 20 --warmup 5 > $O/r2j_bench_cfg3.json 2> $O/r2j_bench_cfg3.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/r2j_ref_cfg3.json 2> $O/r2j_ref_cfg3.err
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/r2j_bench_cfg2.json 2> $O/r2j_bench_cfg2.err
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/r2j_bench_cfg4.json 2> $O/r2j_bench_cfg4.err
python bench.py --config 5 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > $O/r2j_bench_cfg5_n4096.json 2> $O/r2j_bench_cfg5.err
timeout 900 python tools/bench_rows.py > $O/r2j_rows.jsonl 2> $O/r2j_rows.err
echo done
