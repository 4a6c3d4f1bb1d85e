python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "conv or edge or backward or guard" 2>&1 | tail -2
timeout 900 python tools/bench_rows.py --rows f1 > gpurun_out/r2j_rows_f1.jsonl 2> gpurun_out/r2j_rows_f1.err; echo rows rc=$?
