"""Eager steps of bench.py's workload (construction + forward chain) for profilers:
python tools/prof_step.py CONFIG STEPS  (ncu launch lists / --set full captures of one step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_13776_b200 as orth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
W = bench.Workload(orth, torch, cfg, 2048, 64, 0, 1, False, "bf16", 0)
for _ in range(steps):
    W.construct()
    W.forward()
torch.cuda.synchronize()
W.plan.check()
print("ok", W.plan.launches)
