python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_ws -c 1 -o gpurun_out/ws_full python tools/conv_one.py 256 256 3 1 1 1 circular 14 256 > gpurun_out/ws_ncu.log 2>&1
echo ncu rc=$?
