python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "64_channel_forms" 2>&1 | tail -2
ORTH_NVCC_FLAGS="-DORTH_CONV_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== plain"; ORTH_CONV_NO_SWAP=1 timeout 120 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 2>&1 | grep "MMA thread\|conv_pad\|CTA timeline" | tail -3
echo "== swap"; timeout 120 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 2>&1 | grep "MMA thread\|conv_pad\|CTA timeline" | tail -3
