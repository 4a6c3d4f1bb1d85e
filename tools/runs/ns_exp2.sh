ORTH_NVCC_FLAGS="-DORTH_NSP_TRACE -DORTH_NS_EXP2" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ORTH_NS_TRACE=1 python tools/ns_trace_one.py dense 2>&1 | grep -A8 "ns_flow:" | tail -8
