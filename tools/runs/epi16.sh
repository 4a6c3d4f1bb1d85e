python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "64 64 3 1 1 1 circular 56 256" "64 64 3 1 1 1 zeros 56 256" "64 64 3 1 1 1 circular 112 64"; do timeout 120 python tools/conv_one.py $L; done
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or edge" 2>&1 | tail -2
