python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 --zeros
python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
python tools/conv_one.py 256 256 3 1 1 1 circular 14 256 --zeros
python tools/conv_one.py 128 128 3 1 1 1 circular 28 256
python tools/conv_one.py 128 128 3 1 1 1 circular 28 256 --zeros
