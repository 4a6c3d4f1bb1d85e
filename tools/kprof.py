"""Live per-kernel GPU time of the bench step (torch.profiler / CUPTI, warm
caches, no serialisation): python tools/kprof.py [config] [steps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
W = bench.build_workload(orth, torch, configs.CONFIGS[cfg](), 0, 1, 0, "bf16", configs.BATCH[cfg],
                         chain=configs.CHAIN[cfg], cfg_id=cfg)
for _ in range(3):
    bench.run_step(W, orth, torch, 1, None)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        bench.run_step(W, orth, torch, 1, None)
    torch.cuda.synchronize()
rows = []
for e in prof.key_averages():
    t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
    if t > 0:
        rows.append((t / steps, e.count / steps, e.key))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"{'us/step':>9} {'calls':>6}  kernel   (sum {tot:.1f} us/step)")
for t, c, k in rows[:30]:
    print(f"{t:9.1f} {c:6.1f}  {k[:100]}")
