timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_certify.py -x -q 2>&1 | tail -2
for c in 2 3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/nsip_$c.json 2>/dev/null; done
timeout 300 python bench.py --config 5 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nsip_5.json 2>/dev/null
python - <<'P'
import json
for c in (2,3,5):
    d=json.loads(open('gpurun_out/nsip_%d.json'%c).read().strip().splitlines()[-1])
    print(c, round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['ms_per_step'],4) for k,v in d['kernel_groups_ms'].items() if k in ('ns','compose','power','scale')})
P
