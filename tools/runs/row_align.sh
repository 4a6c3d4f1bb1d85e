for al in 1 8; do
  ORTH_CONV_ROW_ALIGN=$al timeout 60 python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
  ORTH_CONV_ROW_ALIGN=$al timeout 60 python tools/conv_one.py 64 64 3 1 1 1 zeros 56 256
done
ORTH_CONV_ROW_ALIGN=8 timeout 600 python -m pytest tests/test_gpu_parity.py -k "forward_and_transpose" -x -q 2>&1 | tail -2
