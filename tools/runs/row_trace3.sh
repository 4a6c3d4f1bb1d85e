ORTH_NVCC_FLAGS="-DORTH_CONV_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 2>&1 | grep -A1 "conv_pad" | tail -2
ORTH_CONV_NO_ROW=1 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 2>&1 | grep -A1 "conv_pad" | tail -2
