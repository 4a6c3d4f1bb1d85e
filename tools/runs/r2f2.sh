set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -x -q > $O/r2f2_pytest.txt 2>&1; echo "pytest rc=$?"; tail -1 $O/r2f2_pytest.txt
python bench.py > $O/r2f2_bench_default.json 2> $O/r2f2_bench_default.err; echo "bench rc=$?"
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/r2f2_bench_cfg2.json 2>/dev/null
python - <<'P'
import json
for f in ('r2f2_bench_default','r2f2_bench_cfg2'):
    d=json.loads(open('gpurun_out/%s.json'%f).read().strip().splitlines()[-1])
    print(f, round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])
P
