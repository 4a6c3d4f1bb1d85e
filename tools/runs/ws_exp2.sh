# conv_ws 256@14 with the A gathers or the weight loads compiled out (timing only, wrong results)
for f in "" "-DORTH_CONV_EXP_NOA" "-DORTH_CONV_EXP_NOB" "-DORTH_CONV_EXP_NOA -DORTH_CONV_EXP_NOB"; do
  ORTH_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "== $f: $(timeout 120 python tools/conv_one.py 256 256 3 1 1 1 circular 14 256 | awk '{print $(NF-1)}') us (256@14), $(timeout 120 python tools/conv_one.py 512 512 3 1 1 1 circular 7 256 | awk '{print $(NF-1)}') us (512@7)"
done
