# conv_ws MMA-thread breakdown after the uniform-issue change (trace build; times inflated ~10%)
ORTH_NVCC_FLAGS="-DORTH_CONV_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "256 256 3 1 1 1 circular 14 256" "128 128 3 1 1 1 circular 28 256" "512 512 3 1 1 1 circular 7 256"; do
  echo "== $L"; timeout 120 python tools/conv_one.py $L 2>&1 | grep "conv_ws\|conv_stack\|stack" | tail -2
done
