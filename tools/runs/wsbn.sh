# conv_ws tile width: N = 256 (4 stages of 48 KB) vs N = 128 (6 stages of 32 KB, the A rows gathered twice)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "256 256 3 1 1 1 circular 14 256" "512 512 3 1 1 1 circular 7 256" "128 256 3 2 1 1 circular 28 256"; do
  for b in 256 128; do echo "$L bn<=$b: $(ORTH_CONV_WS_BN=$b timeout 120 python tools/conv_one.py $L | awk '{print $(NF-1)}')"; done
done
echo "== bench bn<=128"; ORTH_CONV_WS_BN=128 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
