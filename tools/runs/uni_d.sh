# uniform MMA issue in conv_ws / conv_pad ROW (two issuers) / conv_stack: layer timings, conv parity, cfg3 bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "64 64 3 1 1 1 circular 56 256" "128 128 3 1 1 1 circular 28 256" "256 256 3 1 1 1 circular 14 256" "512 512 3 1 1 1 circular 7 256" "256 256 3 1 2 8 zeros 14 256"; do timeout 120 python tools/conv_one.py $L; done
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or edge or backward" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['unit'], d['ms_per_step'], d.get('e2e',{}).get('value'))"
