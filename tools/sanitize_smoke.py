"""A small workload that reaches every kernel family once, for compute-sanitizer runs (one tool per
gpurun call): python tools/sanitize_smoke.py.  Small shapes (the sanitizer slows kernels 10-100x)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs  # noqa: E402
from tests.helpers import pack_params  # noqa: E402


def build(layers, compute, N=2, **kw):
    plan = orth.Plan(layers, 0, compute=compute, max_batch=N, **kw)
    params, _ = pack_params(plan, 5)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    res = torch.zeros(plan.n_matrices, device="cuda")
    plan.orthogonalize(p, ortho, None, res)   # power + NS (flow / persist) + residual
    plan.orthogonalize(p, ortho)               # convergence check from the last Gram
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
    plan.compose(ortho, kf, kb)
    plan.check()
    return plan, p, ortho, kf, kb


def main():
    for compute in ("f32", "bf16"):
        layers = configs.cfg2()[:7] + [dict(kind="conv", c_in=512, c_out=512, k=3, s=1, d=1, g=1,
                                            padding_mode="circular", H=4),
                                       dict(kind="conv", c_in=64, c_out=64, k=3, s=1, d=2, g=2,
                                            padding_mode="zeros", H=12),
                                       dict(kind="convT", c_in=64, c_out=64, k=3, s=2, d=1, g=1,
                                            padding_mode="circular", H=8)]
        plan, p, ortho, kf, kb = build(layers, compute, N=2, vjp=1)
        for l, d in enumerate(layers):
            H = d["H"]
            if d["kind"] == "convT":
                x = torch.randn(2, H, H, d["c_in"], device="cuda").to(torch.bfloat16)
                y = torch.empty(2, H * d["s"], H * d["s"], d["c_out"], device="cuda", dtype=torch.bfloat16)
                plan.conv_transpose(l, plan.kernel_bf16(kb, l), x, y)
                continue
            Ho, Wo = plan.out_hw(l, H, H)
            x = torch.randn(2, H, H, d["c_in"], device="cuda").to(torch.bfloat16)
            y = torch.empty(2, Ho, Wo, d["c_out"], device="cuda", dtype=torch.bfloat16)
            plan.conv_forward(l, plan.kernel_bf16(kb, l), x, y)        # stem / window / gather / split-K
            xt = torch.empty_like(x)
            plan.conv_transpose(l, plan.kernel_bf16(kb, l), y, xt)      # adjoints
            dK = torch.zeros(plan.kernel_shape(l), device="cuda")
            plan.conv_wgrad(l, x, y, dK)                                 # weight gradient
        dortho = torch.zeros_like(p)
        plan.compose_vjp(ortho, torch.randn(plan.kf32_numel, device="cuda"), dortho)
        dparams = torch.zeros_like(p)
        plan.orthogonalize_vjp(p, dortho, dparams)
        plan.certify(3, plan.kernel_f32(kf, 3).reshape(-1).contiguous(), 8, 8, power_iters=5)
        plan.check()
    soc = [dict(kind="soc", c_in=64, c_out=64, k=3, s=1, d=1, g=1, terms=6, padding_mode="circular", H=16)]
    plan, p, ortho, kf, kb = build(soc, "bf16")
    x = torch.randn(2, 16, 16, 64, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    plan.conv_forward(0, plan.kernel_bf16(kb, 0), x, y)              # 13 x 13 gather conv
    plan.conv_transpose(0, plan.kernel_bf16(kb, 0), y, x)
    stem = [dict(kind="conv", c_in=3, c_out=64, k=4, s=4, d=1, g=1, padding_mode="circular", H=32)]
    plan, p, ortho, kf, kb = build(stem, "bf16")
    x = torch.randn(3, 32, 32, 3, device="cuda").to(torch.bfloat16)
    dy = torch.randn(3, 8, 8, 64, device="cuda").to(torch.bfloat16)
    nb = orth.orth_conv_wgrad_workspace(plan.h, 0, 3, 32, 32, orth.BF16)
    ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
    plan.conv_wgrad(0, x, dy, torch.zeros(plan.kernel_shape(0), device="cuda"), workspace=ws)   # small SIMT
    plan.certify(0, plan.kernel_f32(kf, 0).reshape(-1).contiguous(), 8, 8, power_iters=3)
    plan.check()
    blk = [dict(kind="conv", c_in=16, c_out=16, k=2, s=1, d=1, g=1, padding_mode="circular", H=8),
           dict(kind="sll", c_in=16, c_out=16, k=2, s=1, d=1, g=1, padding_mode="circular", H=8),
           dict(kind="conv", c_in=16, c_out=32, k=3, s=2, d=1, g=1, padding_mode="circular", H=8),
           dict(kind="sll_block", c_in=16, c_out=32, k=1, s=2, d=1, g=1, padding_mode="circular", H=8,
                pre=0, sll=1, post=2)]
    plan, p, ortho, kf, kb = build(blk, "bf16")
    x = torch.randn(2, 8, 8, 16, device="cuda").to(torch.bfloat16)
    y = torch.empty(2, 4, 4, 32, device="cuda", dtype=torch.bfloat16)
    plan.conv_forward(3, plan.block_kernels(kb, 3)[0].reshape(-1), x, y, bias=torch.zeros(16, device="cuda"))
    plan.check()
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
