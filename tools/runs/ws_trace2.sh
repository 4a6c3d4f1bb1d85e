for f in "-DORTH_CONV_TRACE" "-DORTH_CONV_TRACE -DORTH_CONV_EXP_NOA" "-DORTH_CONV_TRACE -DORTH_CONV_EXP_NOB" "-DORTH_CONV_TRACE -DORTH_CONV_EXP_NOA -DORTH_CONV_EXP_NOB"; do
  ORTH_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "== $f"; python tools/conv_one.py 256 256 3 1 1 1 circular 14 256 2>&1 | grep conv_ws | tail -1
done
