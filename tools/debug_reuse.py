"""Compare the shifted-copy reuse conv path against the per-tap gather path
(ORTH_CONV_NO_REUSE is read once per process, so each path runs in its own
subprocess) and report where they differ."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CODE = r'''
import sys, numpy as np, torch
import paper_2601_13776_b200 as orth
ci, co, k, d, H, W, mode = [int(a) if a.isdigit() else a for a in sys.argv[1:8]]
layer = dict(kind="conv", c_in=ci, c_out=co, k=k, s=1, d=d, g=1, padding_mode=mode)
plan = orth.Plan([layer], 0)
g = torch.Generator().manual_seed(1)
K = (torch.randn((co, k, k, ci), generator=g) / (ci * k * k) ** 0.5).to(torch.bfloat16).cuda()
x = torch.randn((1, H, W, ci), generator=g).to(torch.bfloat16).cuda()
Ho, Wo = plan.out_hw(0, H, W)
y = torch.zeros((1, Ho, Wo, co), device="cuda", dtype=torch.bfloat16)
plan.conv_forward(0, K, x, y)
torch.cuda.synchronize()
np.save(sys.argv[8], y.float().cpu().numpy())
'''

args = sys.argv[1:] or ["64", "64", "3", "1", "10", "10", "circular"]
outs = []
for tag, env in (("reuse", {}), ("gather", {"ORTH_CONV_NO_REUSE": "1"})):
    f = f"/tmp/dbg_{tag}.npy"
    subprocess.run([sys.executable, "-c", CODE, *args, f], check=True, env={**os.environ, **env})
    outs.append(f)
import numpy as np  # noqa: E402
a, b = np.load(outs[0]), np.load(outs[1])
err = np.abs(a - b).max(axis=-1)[0]
print("shape", a.shape, "max abs diff", np.abs(a - b).max())
np.set_printoptions(linewidth=200, precision=2, suppress=True)
print(err)
