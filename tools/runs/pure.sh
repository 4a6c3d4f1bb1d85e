for f in "-DORTH_ROW_EXP_FILL=1" "-DORTH_ROW_EXP_FILL=1 -DORTH_ROW_EXP_VERBATIM"; do
ORTH_NVCC_FLAGS="-DORTH_ROW_EXP_PURE -DORTH_ROW_EXP_NOB $f -DORTH_CONV_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== PURE NOB $f"; python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 2>&1 | grep "MMA thread\|CTA timeline" | tail -2
done
