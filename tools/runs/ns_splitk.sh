timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py tests/test_gpu_certify.py -x -q 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export ORTH_NS_NO_SPLITK=1; fi
  for c in 2 3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/nssk_${c}_$v.json 2>/dev/null; done
done
python - <<'P'
import json
for v in (0,1):
  for c in (2,3):
    d=json.loads(open('gpurun_out/nssk_%d_%d.json'%(c,v)).read().strip().splitlines()[-1])
    print('nosplit' if v else 'split', c, round(d['value'],1), round(d['ms_per_step'],3), {k: round(v2['ms_per_step'],4) for k,v2 in d['kernel_groups_ms'].items() if k in ('ns','compose')})
P
