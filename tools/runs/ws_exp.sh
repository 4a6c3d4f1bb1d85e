python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
ORTH_NVCC_FLAGS=-DORTH_CONV_EXP_NOA python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo NOA; python tools/conv_one.py 256 256 3 1 1 1 circular 14 256; python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
ORTH_NVCC_FLAGS=-DORTH_CONV_EXP_NOB python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo NOB; python tools/conv_one.py 256 256 3 1 1 1 circular 14 256; python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
ORTH_NVCC_FLAGS="-DORTH_CONV_EXP_NOA -DORTH_CONV_EXP_NOB" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo NOA+NOB; python tools/conv_one.py 256 256 3 1 1 1 circular 14 256; python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
