timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_soc.py tests/test_gpu_sll.py tests/test_gpu_backward.py tests/test_gpu_fullsize.py tests/test_gpu_certify.py -x -q 2>&1 | tail -2
for c in 2 3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cmpnof_$c.json 2>/dev/null; done
python - <<'P'
import json
for c in (2,3):
    d=json.loads(open('gpurun_out/cmpnof_%d.json'%c).read().strip().splitlines()[-1])
    print(c, round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['ms_per_step'],4) for k,v in d['kernel_groups_ms'].items() if k in ('ns','compose','emit')})
P
