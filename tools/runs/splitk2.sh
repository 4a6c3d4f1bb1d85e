timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_guard.py -k "splitk or forward_and_transpose or cfg3 or guard or replay" -x -q 2>&1 | tail -2
python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
ORTH_CONV_NO_SPLITK=1 python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/splitk2.json 2>/dev/null
python - <<'P'
import json
d=json.loads(open('gpurun_out/splitk2.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['ms_per_step'],3), [round(x*1000) for x in d['breakdown']['conv_per_layer_ms']])
P
