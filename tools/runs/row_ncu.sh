python tools/conv_one.py 64 64 3 1 1 1 circular 56 256
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_pad -c 1 -o gpurun_out/row_full python tools/conv_one.py 64 64 3 1 1 1 circular 56 256 > gpurun_out/row_ncu.log 2>&1
echo ncu rc=$?
