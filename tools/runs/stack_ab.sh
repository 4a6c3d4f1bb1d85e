# conv_stack (stacked TMA windows) vs conv_ws (gathered rows) for the layers stack_rule picks, after the issuer rewrite
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "128 128 3 1 1 1 circular 28 256" "128 128 3 1 1 1 zeros 28 256" "64 128 3 2 1 1 circular 56 256" "128 128 3 1 1 1 circular 16 256"; do
  for adj in "" "--adjoint"; do
    s=$(timeout 120 python tools/conv_one.py $L $adj | awk '{print $(NF-1)}')
    w=$(ORTH_CONV_NO_STACK=1 timeout 120 python tools/conv_one.py $L $adj | awk '{print $(NF-1)}')
    echo "$L $adj: stack $s ws $w"
  done
done
echo "== bench NO_STACK"; ORTH_CONV_NO_STACK=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
