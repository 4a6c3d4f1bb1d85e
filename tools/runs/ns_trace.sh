ORTH_NVCC_FLAGS=-DORTH_NSP_TRACE python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in dense dense4 cfg2; do echo "=== $w"; ORTH_NS_TRACE=1 python tools/ns_trace_one.py $w 2>&1 | grep -A12 "ns_flow:" | head -40; done
