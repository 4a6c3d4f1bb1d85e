python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in "64 128 3 2 1 1 circular 56 256" "64 128 3 2 1 1 zeros 56 256" "128 256 3 2 1 1 circular 28 256" "256 512 3 2 1 1 circular 14 256"; do timeout 60 python tools/conv_one.py $L --adjoint; done
timeout 1200 python -m pytest tests -m gpu -x -q -k "conv or edge or backward" 2>&1 | tail -2
