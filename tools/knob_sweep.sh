#!/bin/bash
# One-GPU A/B sweep of the plan's env knobs on the default cfg2 bench (value = layers/s).
mkdir -p gpurun_out
out=gpurun_out/knob_sweep.txt; : > $out
run() { v=$(env "$@" timeout 240 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), d['breakdown_ms'])"); echo "$* :: $v" >> $out; }
run BASE=1
for kv in ORTH_CONV_PAIR=1 ORTH_POWER_CTAS_PER_SM=2 ORTH_POWER_CTAS_PER_SM=8 ORTH_NS_W64_MIN=16 ORTH_NS_W64_MIN=64 \
          ORTH_NS_FULLGRAM_MIN=256 ORTH_NS_FULLGRAM_MIN=1024 ORTH_STEM_CTAS_PER_SM=4 ORTH_STEM_CTAS_PER_SM=8 ORTH_CONV_STACK=1 ORTH_NS_MODE=sync; do
  run $kv
done
run BASE=2
