#!/bin/bash
set -u
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2j_launches_cfg3.csv \
    python tools/prof_step.py 3 2 > $O/r2j_launches_cfg3.log 2>&1
echo "ncu rc=$?"
