# per-phase tap counts precomputed on the host (no tap_valid modulo arithmetic in the MMA issuer per tile)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "64 128 3 2 1 1 circular 56 256" "128 256 3 2 1 1 circular 28 256" "256 256 3 1 1 1 circular 14 256" "512 512 3 1 1 1 circular 7 256"; do
  timeout 60 python tools/conv_one.py $L; timeout 60 python tools/conv_one.py $L --adjoint
done
timeout 1200 python -m pytest tests -m gpu -x -q -k "conv or edge or backward or guard" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['ms_per_step'], d['kernel_groups_ms']['conv_ws<256>']['ms_per_step'])"
