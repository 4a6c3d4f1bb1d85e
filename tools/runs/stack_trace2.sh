ORTH_NVCC_FLAGS="-DORTH_STACK_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "128 128 3 1 1 1 circular 28 256" "128 128 3 1 1 1 circular 16 256"; do echo "== $L"; timeout 120 python tools/conv_one.py $L 2>&1 | grep "conv_stack\|fwd" | tail -2; done
