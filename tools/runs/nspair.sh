# NS flow: two K blocks per stage (one issuer wait per 8 MMAs) for single-pass phases
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "construction or ns or parity_tensor or determinism or not_converged or status or fullsize" 2>&1 | tail -2
for c in 2 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['kernel_groups_ms']; print('cfg', d['config']['workload'][:8], d['value'], d['ms_per_step'], 'ns', g['ns']['ms_per_step'], 'compose', g['compose']['ms_per_step'], 'roof', d['roofline']['frac'])"; done
