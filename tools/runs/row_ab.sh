python -m pytest tests/test_gpu_parity.py -k "forward_and_transpose" -x -q 2>&1 | tail -3
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
ORTH_CONV_NO_ROW=1 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
python tools/conv_one.py 64 64 3 1 1 1 zeros 56 256
ORTH_CONV_NO_ROW=1 python tools/conv_one.py 64 64 3 1 1 1 zeros 56 256
python tools/conv_one.py 64 64 3 1 1 1 circular 32 256
ORTH_CONV_NO_ROW=1 python tools/conv_one.py 64 64 3 1 1 1 circular 32 256
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 --adjoint
ORTH_CONV_NO_ROW=1 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 --adjoint
