# conv_pad one-MMA-chain-per-tap issuers (plain / swapped) after the uniform rewrite, vs the kernel-row form
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
L="64 64 3 1 1 1 circular 56 256"
echo "row";   timeout 120 python tools/conv_one.py $L
echo "swap";  ORTH_CONV_NO_ROW=1 timeout 120 python tools/conv_one.py $L
echo "plain"; ORTH_CONV_NO_ROW=1 ORTH_CONV_NO_SWAP=1 timeout 120 python tools/conv_one.py $L
echo "plain zeros"; ORTH_CONV_NO_ROW=1 ORTH_CONV_NO_SWAP=1 timeout 120 python tools/conv_one.py 64 64 3 1 1 1 zeros 56 256
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or edge or backward" 2>&1 | tail -2
ORTH_CONV_NO_ROW=1 ORTH_CONV_NO_SWAP=1 timeout 900 python -m pytest tests -m gpu -x -q -k "conv and parity" 2>&1 | tail -2
