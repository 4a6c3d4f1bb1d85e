"""Run the cfg2 construction (orthogonalize + compose) a few times: a short
command for ncu captures of the construction kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs  # noqa: E402
from tests.helpers import pack_params  # noqa: E402

compute = sys.argv[1] if len(sys.argv) > 1 else "bf16"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
plan = orth.Plan(configs.cfg2(), 0, compute=compute)
params, _ = pack_params(plan, 2)
p = torch.from_numpy(params).cuda()
o = torch.zeros_like(p)
kf = torch.zeros(plan.kf32_numel, device="cuda")
kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    plan.orthogonalize(p, o)
    plan.compose(o, kf, kb)
plan.check()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
plan.orthogonalize(p, o)
e.record()
torch.cuda.synchronize()
print(f"orthogonalize {s.elapsed_time(e):.3f} ms")
