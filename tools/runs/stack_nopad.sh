timeout 900 python -m pytest tests/test_gpu_parity.py -k "forward_and_transpose or stack or splitk" -x -q 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_guard.py tests/test_gpu_edges.py -x -q 2>&1 | tail -1
python tools/conv_one.py 128 128 3 1 1 1 circular 28 256
python tools/conv_one.py 128 128 3 1 1 1 zeros 28 256
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stack_nopad.json 2>/dev/null
python - <<'P'
import json
d=json.loads(open('gpurun_out/stack_nopad.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['ms_per_step'],3), [round(x*1000) for x in d['breakdown']['conv_per_layer_ms']])
P
