set -u
run() {
python tools/conv_one.py 256 256 4 2 1 1 circular 32 256
python tools/conv_one.py 128 256 3 2 1 1 circular 32 256
python tools/conv_one.py 64 128 3 2 1 1 circular 56 256
python tools/conv_one.py 256 256 3 1 1 1 circular 14 256
python tools/conv_one.py 256 512 3 2 1 1 circular 14 256
}
echo NEW; run
cp gpurun_in/conv_tc_old.cu paper_2601_13776_b200/csrc/conv_tc.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo OLD; run
