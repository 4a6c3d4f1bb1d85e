# uniform-register ROW MMA issue: timing + conv parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
python tools/conv_one.py 64 64 3 1 1 1 zeros 56 256
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or edge" 2>&1 | tail -3
