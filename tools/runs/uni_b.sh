B="-DORTH_CONV_TRACE -DORTH_ROW_EXP_NOA -DORTH_ROW_EXP_NOEPI"
for f in "-DORTH_ROW_EXP_NOWAIT_T" "-DORTH_ROW_EXP_NOWAIT_A" "-DORTH_ROW_EXP_NOWAIT_T -DORTH_ROW_EXP_NOWAIT_A" "-DORTH_ROW_EXP_NOWAIT_T -DORTH_ROW_EXP_NOWAIT_A -DORTH_ROW_EXP_NOCOMMIT_T"; do
ORTH_NVCC_FLAGS="$B $f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== $f"; python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 2>&1 | grep "MMA thread" | tail -1
done
