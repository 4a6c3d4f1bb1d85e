python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ns_flow -c 1 -o gpurun_out/nsflow_dense python tools/ns_trace_one.py dense > gpurun_out/nsflow_ncu.log 2>&1
echo rc=$?
