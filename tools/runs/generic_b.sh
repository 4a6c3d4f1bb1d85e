# kernel-row vs swapped vs plain (one MMA chain per tap) for the 64-channel layers, forward + adjoint, and cfg3 end to end
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "64 64 3 1 1 1 circular 56 256" "64 64 3 1 1 1 zeros 56 256" "64 64 3 1 1 1 circular 32 256" "32 64 3 1 1 1 circular 32 256"; do
  for adj in "" "--adjoint"; do
    r=$(timeout 120 python tools/conv_one.py $L $adj | awk '{print $NF, $(NF-1)}')
    s=$(ORTH_CONV_NO_ROW=1 timeout 120 python tools/conv_one.py $L $adj | awk '{print $(NF-1)}')
    p=$(ORTH_CONV_NO_ROW=1 ORTH_CONV_NO_SWAP=1 timeout 120 python tools/conv_one.py $L $adj | awk '{print $(NF-1)}')
    echo "$L $adj: row $r swap $s plain $p"
  done
done
for v in "" "ORTH_CONV_NO_ROW=1" "ORTH_CONV_NO_ROW=1 ORTH_CONV_NO_SWAP=1"; do
  echo "== bench $v"; env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
