timeout 900 python -m pytest tests/test_gpu_parity.py -k "construction or tensor_core or determinism or frobenius or not_converged" -x -q 2>&1 | tail -2
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ns3d_on.json 2>/dev/null
ORTH_NS_NO_TMA3D=1 timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ns3d_off.json 2>/dev/null
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ns3d_on3.json 2>/dev/null
python - <<'P'
import json
for f in ('ns3d_on','ns3d_off','ns3d_on3'):
    d=json.loads(open('gpurun_out/%s.json'%f).read().strip().splitlines()[-1])
    print(f, d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],4) for k,v in d['kernel_groups_ms'].items() if k in ('ns','compose','power')})
P
