python tools/conv_one.py 128 128 3 1 1 1 circular 28 256
ORTH_CONV_PAD_COMAX=128 ORTH_CONV_NO_STACK=1 python tools/conv_one.py 128 128 3 1 1 1 circular 28 256
ORTH_CONV_NO_STACK=1 python tools/conv_one.py 128 128 3 1 1 1 circular 28 256
python tools/conv_one.py 128 128 3 1 1 1 zeros 28 256
ORTH_CONV_PAD_COMAX=128 ORTH_CONV_NO_STACK=1 python tools/conv_one.py 128 128 3 1 1 1 zeros 28 256
