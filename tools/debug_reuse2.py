"""Single-tap probe of the reuse conv path: for each tap t, weights nonzero at
t only; report which tap / shift of the gather path the output matches."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import sys, numpy as np, torch
import paper_2601_13776_b200 as orth
k, H, W = 3, 10, 10
layer = dict(kind="conv", c_in=64, c_out=64, k=k, s=1, d=1, g=1, padding_mode="circular")
plan = orth.Plan([layer], 0)
g = torch.Generator().manual_seed(1)
x = torch.randn((1, H, W, 64), generator=g).to(torch.bfloat16).cuda()
res = []
for t in range(k * k):
    K = torch.zeros((64, k, k, 64))
    K[:, t // k, t % k, :] = torch.eye(64)
    y = torch.zeros((1, H, W, 64), device="cuda", dtype=torch.bfloat16)
    plan.conv_forward(0, K.to(torch.bfloat16).cuda(), x, y)
    res.append(y.float().cpu().numpy()[0])
np.save(sys.argv[1], np.stack(res))
np.save(sys.argv[1] + ".x.npy", x.float().cpu().numpy()[0])
'''
outs = []
for tag, env in (("reuse", {}), ("gather", {"ORTH_CONV_NO_REUSE": "1"})):
    f = f"/tmp/dbg2_{tag}.npy"
    subprocess.run([sys.executable, "-c", CODE, f], check=True, env={**os.environ, **env})
    outs.append(f)
import numpy as np  # noqa: E402
R, G = np.load(outs[0]), np.load(outs[1])
x = np.load(outs[0] + ".x.npy")
for t in range(9):
    match = [u for u in range(9) if np.abs(R[t] - G[u]).max() < 1e-3]
    found = None
    for dy in range(-3, 4):
        for dx in range(-3, 4):
            if np.abs(R[t] - np.roll(np.roll(x, -dy, 0), -dx, 1)).max() < 1e-3:
                found = (dy, dx)
    print("tap", t, "matches gather taps", match, "equals x shifted by", found, "max", np.abs(R[t]).max())
