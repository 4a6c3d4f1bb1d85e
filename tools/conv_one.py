"""Time one conv layer (forward, or --adjoint) on the GPU: python tools/conv_one.py ci co k s d g mode H [N] [--adjoint].
Random BF16 kernel/activations (timing only); prints the mean of 20 launches in us."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
ci, co, k, s, d, g = map(int, args[:6])
mode, H = args[6], int(args[7])
N = int(args[8]) if len(args) > 8 else 256
adj = "--adjoint" in sys.argv
zeros = "--zeros" in sys.argv   # all-zero operands: separates data-dependent (power) effects from the schedule
layer = dict(kind="conv", c_in=ci, c_out=co, k=k, s=s, d=d, g=g, padding_mode=mode, grid=(H, H))
plan = orth.Plan([layer], 0, max_batch=N)
kb = (torch.randn(co, k, k, ci // g, device="cuda") * 0.05).to(torch.bfloat16)
x = torch.randn(N, H, H, ci, device="cuda").to(torch.bfloat16)
Ho, Wo = plan.out_hw(0, H, H)
y = torch.randn(N, Ho, Wo, co, device="cuda").to(torch.bfloat16)
if zeros:
    kb.zero_(); x.zero_(); y.zero_()
f = (lambda: plan.conv_transpose(0, kb, y, x)) if adj else (lambda: plan.conv_forward(0, kb, x, y))
for _ in range(3):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    f()
e1.record()
torch.cuda.synchronize()
plan.check()
plan.trace(True)   # one traced call: which kernel variant ran
f()
torch.cuda.synchronize()
recs = plan.trace_read()
plan.trace(False)
variant = recs[-1]["variant"] if recs else "?"
print(f"{' '.join(args)} {'adj' if adj else 'fwd'}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us  [{variant}]")
