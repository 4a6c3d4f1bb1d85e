"""f1: backward of the path on the GPU against the float64
oracle VJPs (oracle/orth_oracle.py: conv2d_wgrad, layer_kernel_vjp,
orthogonalize_vjp -- pinned by torch, the bilinear identity and finite
differences in test_oracle_pins.py).

* weight gradient: orth_conv_wgrad (tcgen05 MN-major GEMM over pixel splits,
  fixed-order reduction; FP32 SIMT) for strided / dilated / grouped / circular /
  zero-padded / transposed layers, elementwise-bounded against the oracle on
  the same BF16 inputs, and the bilinear identity at full size."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from tests.helpers import nchw, oracle_layer, rel

pytestmark = pytest.mark.gpu

WG_CASES = [  # (ci, co, k, s, d, g, mode, H, kind, N)
    (64, 64, 3, 1, 1, 1, "circular", 8, "conv", 3), (128, 256, 3, 2, 1, 1, "circular", 16, "conv", 2),
    (256, 128, 3, 1, 1, 1, "zeros", 7, "conv", 3), (64, 128, 3, 1, 2, 2, "circular", 12, "conv", 2),
    (1024, 1024, 3, 1, 2, 32, "circular", 8, "conv", 2), (96, 80, 3, 2, 1, 1, "zeros", 9, "conv", 2),
    (64, 64, 3, 2, 1, 1, "circular", 8, "convT", 2), (512, 512, 3, 1, 1, 1, "circular", 4, "conv", 16),
    (3, 64, 4, 4, 1, 1, "circular", 16, "conv", 2), (16, 16, 5, 1, 1, 1, "zeros", 9, "conv", 2),
]


@pytest.mark.parametrize("case", WG_CASES)
@pytest.mark.parametrize("io", ["bf16", "f32"])
def test_conv_wgrad(cuda_lib, case, io):
    ci, co, k, s, d, g, mode, H, kind, N = case
    layer = dict(kind=kind, c_in=ci, c_out=co, k=k, s=s, d=d, g=g, padding_mode=mode)
    plan = cuda_lib.Plan([layer], 0)
    OL = oracle_layer(layer)
    ci_f, co_f = OL.fwd_channels()
    Hb = H * s if kind == "convT" else H
    Ho, Wo = plan.out_hw(0, Hb, Hb)
    x = gen.activations((N, Hb, Hb, ci_f), (81, 1, ci, co, 6))
    dy = gen.activations((N, Ho, Wo, co_f), (81, 2, ci, co, 6))
    dt = torch.bfloat16 if io == "bf16" else torch.float32
    if io == "bf16":
        x, dy = gen.bf16_round(x), gen.bf16_round(dy)
    kshape = plan.kernel_shape(0)
    dK = torch.full(kshape, float("nan"), device="cuda")
    plan.conv_wgrad(0, torch.from_numpy(x).cuda().to(dt), torch.from_numpy(dy).cuda().to(dt), dK)
    plan.check()
    got = dK.cpu().numpy().astype(np.float64)
    x64, dy64 = nchw(x.astype(np.float64)), nchw(dy.astype(np.float64))
    ref = O.conv2d_wgrad(x64, dy64, kshape, s=s, d=d, g=g, mode=mode)
    absref = O.conv2d_wgrad(np.abs(x64), np.abs(dy64), kshape, s=s, d=d, g=g, mode=mode)
    # products of BF16 (or FP32) inputs are exact in FP32; the only error is FP32 accumulation
    err = np.abs(got - ref)
    assert (err <= 2.0 ** -16 * absref + 1e-30).all(), (float((err / (absref + 1e-30)).max()))
    assert rel(got, ref) < 1e-5
