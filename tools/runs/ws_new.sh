timeout 900 python -m pytest tests/test_gpu_parity.py -k "forward_and_transpose or splitk" -x -q 2>&1 | tail -2
python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
python tools/conv_one.py 128 256 3 2 1 1 circular 28 256
python tools/conv_one.py 64 128 3 2 1 1 circular 56 256
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ws_new.json 2>/dev/null
python - <<'P'
import json
d=json.loads(open('gpurun_out/ws_new.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['ms_per_step'],3), d['roofline']['kernel'], round(d['roofline']['frac'],3), [round(x*1000) for x in d['breakdown']['conv_per_layer_ms']])
P
