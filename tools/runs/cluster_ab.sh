# conv_ws weight multicast across a cluster (ORTH_CONV_CLUSTER) re-measured after the issuer rewrite
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "256 256 3 1 1 1 circular 14 256" "512 512 3 1 1 1 circular 7 256" "128 256 3 2 1 1 circular 28 256"; do
  for c in 1 2 4; do echo "$L cs=$c: $(ORTH_CONV_CLUSTER=$c timeout 120 python tools/conv_one.py $L | awk '{print $(NF-1)}')"; done
done
for c in 2 4; do echo "== bench cs=$c"; ORTH_CONV_CLUSTER=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
