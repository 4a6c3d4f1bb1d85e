ORTH_NVCC_FLAGS="-DORTH_CONV_TRACE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/conv_one.py 64 128 3 2 1 1 circular 56 256 --adjoint > gpurun_out/adj_trace2.txt 2>&1
grep "conv_ws" gpurun_out/adj_trace2.txt | tail -2
