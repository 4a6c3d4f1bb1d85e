"""Out-of-bounds and race guards for every kernel family, in place of compute-sanitizer (closed on the
GPU pool: runs under it left GPUs needing a reset).

* guard bands: every caller-owned buffer an entry point writes (ortho, residuals, FP32 / BF16 kernels,
  activations, dK, VJP outputs, workspaces) is a view into a larger allocation whose margins hold a bit
  pattern; after each call the margins must be bit-identical (a write past either end of any buffer,
  e.g. a ragged tile's epilogue or a split-K partial, trips it);
* unwritten outputs: outputs start as NaN and must come back finite;
* races: the dataflow / persistent kernels (power, NS flow, composition flow, split-K conv, wgrad splits,
  certify) are replayed many times and must be bitwise identical every time (their inter-CTA counters
  and flags order the work; a missing acquire / release shows up as a nondeterministic result)."""
import numpy as np
import pytest
import torch

from synth import configs
from tests.helpers import oracle_layer, pack_params

pytestmark = pytest.mark.gpu

M = 4096   # margin elements on each side


class Guarded:
    def __init__(self, n, dtype, fill=float("nan")):
        self.n = n
        self.big = torch.empty(n + 2 * M, dtype=dtype, device="cuda")
        pat = torch.arange(n + 2 * M, device="cuda") % 251
        self.big.copy_(pat.to(dtype) if dtype == torch.uint8 else (pat - 125.0).to(dtype))
        self.ref = self.big.clone()
        self.t = self.big[M:M + n]
        self.t.fill_(fill)

    def view(self, *shape):
        return self.t.view(*shape) if shape else self.t

    def check(self, what):
        torch.cuda.synchronize()
        a = self.big[:M].view(torch.int8 if self.big.element_size() == 1 else
                              {2: torch.int16, 4: torch.int32, 8: torch.int64}[self.big.element_size()])
        b = self.ref[:M].view(a.dtype)
        c = self.big[M + self.n:].view(a.dtype)
        d = self.ref[M + self.n:].view(a.dtype)
        assert torch.equal(a, b), f"{what}: write before the buffer"
        assert torch.equal(c, d), f"{what}: write past the end of the buffer"


def _construct(orth, layers, compute, N, cfg_id=5, vjp=1):
    plan = orth.Plan(layers, 0, compute=compute, max_batch=N, vjp=vjp)
    params, _ = pack_params(plan, cfg_id)
    p = Guarded(params.size, torch.float32)
    p.view().copy_(torch.from_numpy(params))
    ortho = Guarded(params.size, torch.float32)
    res = Guarded(plan.n_matrices, torch.float32)
    plan.orthogonalize(p.view(), ortho.view(), None, res.view())
    plan.check()
    for g, w in ((p, "params"), (ortho, "ortho"), (res, "residual_out")):
        g.check(f"orthogonalize {w}")
    assert torch.isfinite(ortho.view()).all()
    kf = Guarded(plan.kf32_numel, torch.float32)
    kb = Guarded(plan.kbf16_numel, torch.bfloat16)
    plan.compose(ortho.view(), kf.view(), kb.view())
    plan.check()
    kf.check("compose kernels_f32")
    kb.check("compose kernels_bf16")
    assert torch.isfinite(kf.view()).all() and torch.isfinite(kb.view().float()).all()
    return plan, p, ortho, kf, kb


LAYERS = [  # every conv kernel family: stem, TMA-window (64 ch), stacked window (>= 128), gather (strided,
    # 256-wide, split-K), grouped packed, dilated zeros, transposed, 13 x 13 gather, dense
    dict(kind="conv", c_in=3, c_out=64, k=4, s=4, d=1, g=1, padding_mode="circular", H=64),
    dict(kind="conv", c_in=64, c_out=64, k=3, s=1, d=1, g=1, padding_mode="circular", H=16),
    dict(kind="conv", c_in=64, c_out=128, k=3, s=2, d=1, g=1, padding_mode="circular", H=16),
    dict(kind="conv", c_in=128, c_out=128, k=3, s=1, d=1, g=1, padding_mode="circular", H=8),
    dict(kind="conv", c_in=512, c_out=512, k=3, s=1, d=1, g=1, padding_mode="circular", H=4),
    dict(kind="conv", c_in=256, c_out=256, k=3, s=1, d=2, g=32, padding_mode="circular", H=8),
    dict(kind="conv", c_in=64, c_out=64, k=3, s=1, d=2, g=1, padding_mode="zeros", H=13),
    dict(kind="convT", c_in=64, c_out=64, k=3, s=2, d=1, g=1, padding_mode="circular", H=8),
    dict(kind="conv", c_in=48, c_out=40, k=3, s=2, d=1, g=1, padding_mode="zeros", H=9),
    dict(kind="dense", c_in=96, c_out=64, k=1, s=1, d=1, g=1, padding_mode="circular", H=1),
]


@pytest.mark.parametrize("compute", ["bf16", "f32"])
def test_guard_bands_every_entry_point(cuda_lib, compute):
    orth = cuda_lib
    N = 3
    plan, p, ortho, kf, kb = _construct(orth, LAYERS, compute, N)
    for l, d in enumerate(LAYERS):
        if d["kind"] == "dense":
            continue
        ci_f, co_f = oracle_layer(d).fwd_channels()
        Hx = d["H"] * d["s"] if d["kind"] == "convT" else d["H"]
        Wx = Hx + (1 if d["padding_mode"] == "zeros" else 0)
        Ho, Wo = plan.out_hw(l, Hx, Wx)
        for io in (torch.bfloat16, torch.float32):
            kern = plan.kernel_bf16(kb.view(), l) if io == torch.bfloat16 else plan.kernel_f32(kf.view(), l)
            x = Guarded(N * Hx * Wx * ci_f, io, 0.0)
            x.view().copy_(torch.randn(x.n, device="cuda").to(io))
            y = Guarded(N * Ho * Wo * co_f, io)
            bias = Guarded(co_f, torch.float32, 0.25)
            plan.conv_forward(l, kern, x.view(N, Hx, Wx, ci_f), y.view(N, Ho, Wo, co_f), bias=bias.view())
            plan.check()
            y.check(f"conv_forward layer {l} {io}")
            assert torch.isfinite(y.view().float()).all(), f"conv_forward layer {l} {io}: unwritten outputs"
            xb = Guarded(N * Hx * Wx * ci_f, io)
            plan.conv_transpose(l, kern, y.view(N, Ho, Wo, co_f), xb.view(N, Hx, Wx, ci_f))
            plan.check()
            xb.check(f"conv_transpose layer {l} {io}")
            assert torch.isfinite(xb.view().float()).all(), f"conv_transpose layer {l} {io}: unwritten outputs"
            shape = plan.kernel_shape(l)
            dK = Guarded(int(np.prod(shape)), torch.float32)
            nb = orth.orth_conv_wgrad_workspace(plan.h, l, N, Hx, Wx, orth.BF16 if io == torch.bfloat16 else orth.F32)
            ws = Guarded(max(nb, 16), torch.uint8, 0)
            plan.conv_wgrad(l, x.view(N, Hx, Wx, ci_f), y.view(N, Ho, Wo, co_f), dK.view(*shape), workspace=ws.view())
            plan.check()
            dK.check(f"conv_wgrad layer {l} {io}")
            ws.check(f"conv_wgrad workspace layer {l} {io}")
            assert torch.isfinite(dK.view()).all(), f"conv_wgrad layer {l} {io}: unwritten outputs"
    dK = torch.randn(plan.kf32_numel, device="cuda")
    dortho = Guarded(p.n, torch.float32)
    plan.compose_vjp(ortho.view(), dK, dortho.view())
    plan.check()
    dortho.check("compose_vjp d_ortho")
    dparams = Guarded(p.n, torch.float32)
    plan.orthogonalize_vjp(p.view(), dortho.view(), dparams.view())
    plan.check()
    dparams.check("orthogonalize_vjp d_params")
    assert torch.isfinite(dparams.view()).all()
    for l in (1, 4, 5, 9):
        Hc = 1 if LAYERS[l]["kind"] == "dense" else 8
        nb = orth.orth_certify_workspace(plan.h, l, Hc, Hc)
        ws = Guarded(nb, torch.uint8, 0)
        out = plan.certify(l, plan.kernel_f32(kf.view(), l).reshape(-1).contiguous(), Hc, Hc, power_iters=4,
                           workspace=ws.view())
        plan.check()
        ws.check(f"certify workspace layer {l}")
        assert torch.isfinite(out).all()


def test_guard_bands_soc_and_sll_block(cuda_lib):
    soc = [dict(kind="soc", c_in=64, c_out=64, k=3, s=1, d=1, g=1, terms=6, padding_mode="circular", H=16)]
    plan, p, ortho, kf, kb = _construct(cuda_lib, soc, "bf16", 2, vjp=0)
    x = torch.randn(2, 16, 16, 64, device="cuda").to(torch.bfloat16)
    y = Guarded(x.numel(), torch.bfloat16)
    plan.conv_forward(0, plan.kernel_bf16(kb.view(), 0), x, y.view(2, 16, 16, 64))
    plan.check()
    y.check("SOC 13x13 conv_forward")
    assert torch.isfinite(y.view().float()).all()
    c, cs, co, H = 32, 32, 64, 8
    blk = [dict(kind="conv", c_in=c, c_out=c, k=2, s=1, d=1, g=1, padding_mode="circular", H=H),
           dict(kind="sll", c_in=c, c_out=cs, k=2, s=1, d=1, g=1, padding_mode="circular", H=H),
           dict(kind="conv", c_in=c, c_out=co, k=3, s=2, d=1, g=1, padding_mode="circular", H=H),
           dict(kind="sll_block", c_in=c, c_out=co, k=1, s=2, d=1, g=1, padding_mode="circular", H=H,
                pre=0, sll=1, post=2)]
    plan, p, ortho, kf, kb = _construct(cuda_lib, blk, "bf16", 2, vjp=0)
    x = torch.randn(2, H, H, c, device="cuda").to(torch.bfloat16)
    y = Guarded(2 * (H // 2) ** 2 * co, torch.bfloat16)
    plan.conv_forward(3, plan.block_kernels(kb.view(), 3)[0].reshape(-1), x, y.view(2, H // 2, H // 2, co),
                      bias=torch.zeros(cs, device="cuda"))
    plan.check()
    y.check("SLL block conv_forward")
    assert torch.isfinite(y.view().float()).all()


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_dataflow_replays_bitwise(cuda_lib, cfg_id):
    """Construction (power, NS flow / persist, composition flow, emit) replayed 25 times: bitwise equal."""
    layers = configs.CONFIGS[cfg_id]()
    plan = cuda_lib.Plan(layers, 0, compute="bf16")
    params, _ = pack_params(plan, cfg_id)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
    plan.orthogonalize(p, ortho)
    plan.compose(ortho, kf, kb)
    o0, f0, b0 = ortho.clone(), kf.clone(), kb.clone()
    for _ in range(25):
        ortho.fill_(float("nan"))
        kf.fill_(float("nan"))
        plan.orthogonalize(p, ortho)
        plan.compose(ortho, kf, kb)
        assert torch.equal(ortho, o0) and torch.equal(kf, f0) and torch.equal(kb.view(torch.int16), b0.view(torch.int16))
    plan.check()


def test_splitk_and_wgrad_replays_bitwise(cuda_lib):
    """Split-K conv (flag handshake between K halves) and the wgrad pixel splits replayed: bitwise equal."""
    layer = dict(kind="conv", c_in=512, c_out=512, k=3, s=1, d=1, g=1, padding_mode="circular")
    N, H = 16, 4
    plan = cuda_lib.Plan([dict(layer, grid=(H, H))], 0, max_batch=N)
    k = torch.randn(512, 3, 3, 512, device="cuda").to(torch.bfloat16) * 0.02
    x = torch.randn(N, H, H, 512, device="cuda").to(torch.bfloat16)
    y = torch.empty(N, H, H, 512, device="cuda", dtype=torch.bfloat16)
    xb = torch.empty_like(x)
    dK = torch.empty(plan.kernel_shape(0), device="cuda")
    plan.conv_forward(0, k, x, y)
    plan.conv_transpose(0, k, y, xb)
    plan.conv_wgrad(0, x, y, dK)
    y0, xb0, dK0 = y.clone(), xb.clone(), dK.clone()
    for _ in range(40):
        plan.conv_forward(0, k, x, y)
        plan.conv_transpose(0, k, y, xb)
        plan.conv_wgrad(0, x, y, dK)
        assert torch.equal(y.view(torch.int16), y0.view(torch.int16))
        assert torch.equal(xb.view(torch.int16), xb0.view(torch.int16))
        assert torch.equal(dK, dK0)
    plan.check()
