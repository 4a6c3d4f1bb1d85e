for c in 2 3; do for v in 0 1; do
  if [ $v = 1 ]; then export ORTH_CONV_STACK=1; else unset ORTH_CONV_STACK; fi
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sab_${c}_$v.json 2>/dev/null
done; done
python - <<'P'
import json
for c in (2,3):
  for v in (0,1):
    d=json.loads(open('gpurun_out/sab_%d_%d.json'%(c,v)).read().strip().splitlines()[-1])
    print(c, v, round(d['value']), round(d['ms_per_step'],3), [round(x*1000) for x in d['breakdown']['conv_per_layer_ms']])
P
