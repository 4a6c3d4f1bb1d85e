for sl in 2 3; do
ORTH_NVCC_FLAGS="-DORTH_NSP_TRACE -DORTH_NS_SLOTS=$sl" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "=== slots $sl"; ORTH_NS_TRACE=1 python tools/ns_trace_one.py dense 2>&1 | grep -A3 "ns_flow:" | tail -4
done
