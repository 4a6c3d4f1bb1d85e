# two-issuer, specialised ROW MMA loop: timing + trace + conv parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
timeout 120 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
timeout 120 python tools/conv_one.py 64 64 3 1 1 1 zeros 56 256
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or edge" 2>&1 | tail -3
ORTH_NVCC_FLAGS="-DORTH_CONV_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 2>&1 | grep "MMA thread\|conv_pad" | tail -2
