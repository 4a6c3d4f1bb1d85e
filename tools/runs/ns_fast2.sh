timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -k "cfg5 or construction or tensor_core or determinism or frobenius or not_converged" -x -q 2>&1 | tail -2
timeout 600 python bench.py --config 5 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nsfast_5.json 2>/dev/null
timeout 600 python bench.py --config 5 --n 2048 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nsfast_5b.json 2>/dev/null
python - <<'P'
import json
for f in ('nsfast_5','nsfast_5b'):
    d=json.loads(open('gpurun_out/%s.json'%f).read().strip().splitlines()[-1])
    print(f, round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['kernel'], round(d['roofline']['frac'],3), round(d['roofline']['frac_vs_sustained'],3))
P
