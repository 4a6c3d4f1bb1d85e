# whole-warp elected MMA issue in conv_pad: timing of the ROW / SW / plain conv_pad layers + conv parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
python tools/conv_one.py 128 128 3 1 1 1 circular 28 256
python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or edge or guard" 2>&1 | tail -3
