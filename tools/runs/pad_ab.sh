python tools/conv_one.py 128 128 3 1 1 1 circular 28 256
python tools/conv_one.py 128 128 3 1 1 1 zeros 28 256
python -m pytest tests/test_gpu_parity.py -k "forward_and_transpose" -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pad_kernel -c 3 python tools/conv_one.py 128 128 3 1 1 1 circular 28 256 2>&1 | grep -E "duration|bytes" | head -12
