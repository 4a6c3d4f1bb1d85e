set -u
O=gpurun_out/cexp.txt; : > $O
python -m pytest tests/test_gpu_parity.py -k "conv" -x -q 2>&1 | tail -3 >> $O
for c in "64 64 3 1 1 1 circular 32" "64 64 3 1 1 1 zeros 32" "64 64 3 1 1 1 circular 32 64" "1024 1024 3 1 1 32 circular 56"; do
  echo "$(python tools/conv_one.py $c 2>&1 | tail -1)" >> $O
done
python tools/prof_conv.py 3 >> $O 2>&1
cat $O
