for v in 0 1; do
  if [ $v = 1 ]; then export ORTH_CONV_STACK=1; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stack_ab_$v.json 2>/dev/null
done
python - <<'P'
import json
for v in (0,1):
    d=json.loads(open('gpurun_out/stack_ab_%d.json'%v).read().strip().splitlines()[-1])
    print(v, round(d['value']), round(d['ms_per_step'],3), [round(x*1000) for x in d['breakdown']['conv_per_layer_ms']])
P
