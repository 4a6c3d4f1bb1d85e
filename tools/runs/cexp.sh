set -u
O=gpurun_out/cexp.txt; : > $O
python -m pytest tests/test_gpu_parity.py -k "conv" -x -q 2>&1 | tail -2 >> $O
for c in "128 128 3 1 1 1 circular 16" "256 256 3 1 1 1 circular 8" "512 512 3 1 1 1 circular 4" "512 512 3 1 1 1 circular 7" "256 256 3 1 1 1 circular 14" "128 128 3 1 1 1 circular 28" "1024 1024 3 1 2 1 circular 56"; do
  echo "tma  $(ORTH_NO_PDL=1 python tools/conv_one.py $c 2>&1 | tail -1)" >> $O
  echo "ws   $(ORTH_NO_PDL=1 ORTH_CONV_NO_TMA=1 python tools/conv_one.py $c 2>&1 | tail -1)" >> $O
done
ORTH_NO_PDL=1 python tools/prof_conv.py 3 >> $O 2>&1
ORTH_NO_PDL=1 ORTH_CONV_NO_TMA=1 python tools/prof_conv.py 3 >> $O 2>&1
cat $O
