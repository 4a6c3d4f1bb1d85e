"""cfg2 forward chain (bf16, batch 256) after one construction: a short command
for ncu captures of the conv kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs, gen  # noqa: E402
from tests.helpers import pack_params  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
layers = configs.cfg2()
plan = orth.Plan(layers, 0, compute="bf16", max_batch=256)
params, _ = pack_params(plan, 2)
p = torch.from_numpy(params).cuda()
o = torch.zeros_like(p)
kf = torch.zeros(plan.kf32_numel, device="cuda")
kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
plan.orthogonalize(p, o)
plan.compose(o, kf, kb)
x = torch.from_numpy(gen.activations((256, 32, 32, 3), (2, 0, 0, 0, 6))).cuda().to(torch.bfloat16)
acts, H = [], 32
for l, d in enumerate(layers):
    Ho, _ = plan.out_hw(l, H, H)
    acts.append(torch.empty((256, Ho, Ho, d["c_out"]), device="cuda", dtype=torch.bfloat16))
    H = Ho
ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(layers) + 1)]
for _ in range(reps):
    cur = x
    ev[0].record()
    for l, y in enumerate(acts):
        plan.conv_forward(l, plan.kernel_bf16(kb, l), cur, y)
        ev[l + 1].record()
        cur = y
torch.cuda.synchronize()
plan.check()
print(" ".join(f"{ev[l].elapsed_time(ev[l + 1]) * 1e3:.0f}" for l in range(len(layers))), "us per layer")
