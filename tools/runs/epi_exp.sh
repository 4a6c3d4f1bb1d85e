for f in "" "-DORTH_ROW_EXP_NOSTORE" "-DORTH_ROW_EXP_NOXCH" "-DORTH_ROW_EXP_NOSTORE -DORTH_ROW_EXP_NOXCH"; do
ORTH_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== $f"; timeout 120 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
done
