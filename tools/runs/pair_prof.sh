ORTH_EXPERIMENTAL=1 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pair_build.log 2>&1 || exit 1
python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
ORTH_CONV_PAIR=1 python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
ORTH_CONV_PAIR=1 python tools/conv_one.py 512 512 3 1 1 1 circular 7 256
ORTH_CONV_PAIR=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_pair -c 1 -o gpurun_out/pair_full python tools/conv_one.py 256 256 3 1 1 1 circular 14 256 > gpurun_out/pair_ncu.log 2>&1
echo ncu rc=$?
