timeout 1200 python -m pytest tests/test_gpu_parity.py -k "construction or tensor_core or determinism or frobenius or not_converged or cfg2" -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_guard.py -x -q 2>&1 | tail -2
ORTH_NVCC_FLAGS="-DORTH_NSP_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ORTH_NS_TRACE=1 python tools/ns_trace_one.py dense 2>&1 | grep -A8 "ns_flow:" | tail -8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/nsfast_$c.json 2>/dev/null; done
python - <<'P'
import json
for c in (2,3):
    d=json.loads(open('gpurun_out/nsfast_%d.json'%c).read().strip().splitlines()[-1])
    print(c, round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['ms_per_step'],4) for k,v in d['kernel_groups_ms'].items() if k in ('ns','compose')})
P
