ORTH_NVCC_FLAGS="-DORTH_NSP_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ORTH_NS_TRACE=1 python tools/ns_trace_one.py dense 2>&1 | grep -A8 "ns_flow:" | tail -8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stcg_$c.json 2>/dev/null; done
python - <<'P'
import json
for c in (2,3):
    d=json.loads(open('gpurun_out/stcg_%d.json'%c).read().strip().splitlines()[-1])
    print(c, round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['ms_per_step'],4) for k,v in d['kernel_groups_ms'].items() if k in ('ns','compose')})
P
