set -u
O=gpurun_out/cexp.txt; : > $O
for c in "128 128 3 1 1 1 circular 16" "256 256 3 1 1 1 circular 8" "512 512 3 1 1 1 circular 4" "256 512 3 2 1 1 circular 8" "128 256 3 2 1 1 circular 16"; do
  echo "ws   $(ORTH_NO_PDL=1 python tools/conv_one.py $c 2>&1 | tail -1)" >> $O
  echo "pair $(ORTH_NO_PDL=1 ORTH_CONV_PAIR=1 python tools/conv_one.py $c 2>&1 | tail -1)" >> $O
done
ORTH_NO_PDL=1 python tools/prof_conv.py 3 >> $O 2>&1
ORTH_NO_PDL=1 ORTH_CONV_PAIR=1 python tools/prof_conv.py 3 >> $O 2>&1
cat $O
