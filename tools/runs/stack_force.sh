python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "256 256 3 1 1 1 circular 14 256" "512 512 3 1 1 1 circular 7 256" "256 256 3 1 1 1 zeros 14 256"; do
  timeout 120 python tools/conv_one.py $L; ORTH_CONV_STACK=1 timeout 120 python tools/conv_one.py $L
done
