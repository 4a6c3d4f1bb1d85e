python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
ORTH_NVCC_FLAGS=-DORTH_ROW_EXP_NOEPI python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
