# final state check: full GPU suite, smoke, default bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py 2>/dev/null | tail -1 > gpurun_out/final_bench.json; python -c "import json; d=json.loads(open('gpurun_out/final_bench.json').read()); print('BENCH', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
