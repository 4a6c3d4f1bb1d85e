python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
ORTH_CONV_NO_ROW=1 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
ORTH_CONV_NO_ROW=1 ORTH_CONV_NO_SWAP=1 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
