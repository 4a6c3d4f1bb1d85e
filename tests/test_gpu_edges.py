"""Edge cases of the conv entry points (a6 / a7 / f1) through the C ABI, against the oracle:

* empty batch (N = 0: a rank's empty shard) -- a no-op for forward / adjoint (outputs untouched, NULL
  activations accepted), dK = 0 for the weight gradient;
* degenerate geometry -- 1-pixel images (H = W = 1, zero and circular padding), images no larger than
  the dilated kernel, a single input / output channel, 1 x 1 kernels, stride = kernel size (RKO only),
  even kernels, prime channel counts -- forward and adjoint on both I/O types, elementwise (R18);
* the network's own construction for degenerate layers (c = 1: BCOP projectors of rank 0, R5) feeding
  the conv, checked against the oracle's kernel and conv."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from tests.helpers import assert_elementwise, nchw, nhwc, oracle_layer, rel

pytestmark = pytest.mark.gpu

BF16_ELEM = (2.0 ** -8, 2.0 ** -12)
F32_ELEM = (2.0 ** -20, 2.0 ** -16)


def test_empty_batch_is_a_noop(cuda_lib):
    layer = dict(kind="conv", c_in=64, c_out=64, k=3, s=1, d=1, g=1, padding_mode="circular")
    plan = cuda_lib.Plan([layer], 0)
    k = torch.randn(64, 3, 3, 64, device="cuda").to(torch.bfloat16)
    x = torch.empty(0, 8, 8, 64, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(0, 8, 8, 64, device="cuda", dtype=torch.bfloat16)
    plan.conv_forward(0, k, x, y)
    plan.conv_transpose(0, k, y, x)
    dK = torch.full(plan.kernel_shape(0), 7.0, device="cuda")
    plan.conv_wgrad(0, x, y, dK)
    plan.check()
    assert (dK == 0).all()
    assert cuda_lib.orth_conv_wgrad_workspace(plan.h, 0, 0, 8, 8, cuda_lib.BF16) == 0


EDGE = [  # (ci, co, k, s, d, g, mode, H, W, kind)
    (8, 8, 3, 1, 1, 1, "zeros", 1, 1, "conv"), (8, 8, 3, 1, 1, 1, "circular", 1, 1, "conv"),
    (8, 8, 3, 1, 2, 1, "zeros", 5, 5, "conv"),            # image = dilated kernel extent
    (1, 1, 3, 1, 1, 1, "circular", 6, 6, "conv"), (1, 7, 3, 1, 1, 1, "zeros", 5, 4, "conv"),
    (5, 1, 3, 1, 1, 1, "zeros", 4, 5, "conv"), (13, 11, 1, 1, 1, 1, "zeros", 3, 7, "conv"),
    (2, 8, 2, 2, 1, 1, "circular", 4, 6, "conv"),        # s = k: RKO only
    (3, 12, 4, 4, 1, 1, "zeros", 9, 10, "conv"), (64, 64, 2, 1, 1, 1, "zeros", 3, 3, "conv"),
    (64, 64, 3, 2, 1, 1, "zeros", 1, 1, "conv"), (64, 128, 3, 2, 1, 1, "zeros", 3, 2, "convT"),
    (128, 128, 3, 1, 1, 1, "circular", 1, 3, "conv"), (256, 256, 3, 1, 2, 8, "zeros", 2, 2, "conv"),
]


@pytest.mark.parametrize("case", EDGE)
@pytest.mark.parametrize("io", ["f32", "bf16"])
def test_degenerate_geometry(cuda_lib, case, io):
    ci, co, k, s, d, g, mode, H, W, kind = case
    layer = dict(kind=kind, c_in=ci, c_out=co, k=k, s=s, d=d, g=g, padding_mode=mode)
    OL = oracle_layer(layer)
    ci_f, co_f = OL.fwd_channels()
    if kind == "convT" or mode == "circular":
        H, W = H * s, W * s
    rng = gen.rng(91, ci, co, k, s)
    K = (rng.standard_normal((co_f, ci_f // g, k, k)) / np.sqrt(ci_f // g * k * k)).astype(np.float32)
    N = 2
    x = gen.activations((N, H, W, ci_f), (91, 1, ci, co, H))
    if io == "bf16":
        K, x = gen.bf16_round(K), gen.bf16_round(x)
        kdev, xdev, tdt = torch.from_numpy(np.transpose(K, (0, 2, 3, 1)).copy()).cuda().to(torch.bfloat16), \
            torch.from_numpy(x).cuda().to(torch.bfloat16), torch.bfloat16
    else:
        kdev, xdev, tdt = torch.from_numpy(K).cuda(), torch.from_numpy(x).cuda(), torch.float32
    plan = cuda_lib.Plan([dict(layer, grid=(H, W))], 0, max_batch=N)
    Ho, Wo = plan.out_hw(0, H, W)
    y = torch.full((N, Ho, Wo, co_f), float("nan"), device="cuda", dtype=tdt)
    plan.conv_forward(0, kdev, xdev, y)
    K64, x64 = K.astype(np.float64), nchw(x.astype(np.float64))
    ref = O.conv2d(x64, K64, s=s, d=d, g=g, mode=mode)
    absref = O.conv2d(np.abs(x64), np.abs(K64), s=s, d=d, g=g, mode=mode)
    elem = BF16_ELEM if io == "bf16" else F32_ELEM
    got = y.float().cpu().numpy()
    assert got.shape == nhwc(ref).shape
    assert_elementwise(got, nhwc(ref), nhwc(absref), *elem, what=f"forward {case} {io}")
    yr = gen.activations((N, Ho, Wo, co_f), (91, 3, ci, co, H))
    if io == "bf16":
        yr = gen.bf16_round(yr)
    xb = torch.full((N, H, W, ci_f), float("nan"), device="cuda", dtype=tdt)
    plan.conv_transpose(0, kdev, torch.from_numpy(yr).cuda().to(tdt), xb)
    yr64 = nchw(yr.astype(np.float64))
    refT = O.conv_transpose2d(yr64, K64, H, W, s=s, d=d, g=g, mode=mode)
    absT = O.conv_transpose2d(np.abs(yr64), np.abs(K64), H, W, s=s, d=d, g=g, mode=mode)
    assert_elementwise(xb.float().cpu().numpy(), nhwc(refT), nhwc(absT), *elem, what=f"adjoint {case} {io}")
    dK = torch.full(plan.kernel_shape(0), float("nan"), device="cuda")
    plan.conv_wgrad(0, xdev, torch.from_numpy(yr).cuda().to(tdt), dK)
    plan.check()
    dref = O.conv2d_wgrad(x64, yr64, dK.shape, s=s, d=d, g=g, mode=mode)
    dabs = O.conv2d_wgrad(np.abs(x64), np.abs(yr64), dK.shape, s=s, d=d, g=g, mode=mode)
    err = np.abs(dK.cpu().numpy().astype(np.float64) - dref)
    assert (err <= 2.0 ** -16 * dabs + 1e-30).all()


@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_degenerate_layers_construct_and_apply(cuda_lib, compute):
    """c = 1 (rank-0 projectors), 1 x 1 and s = k layers built by the library, applied by it, vs the oracle."""
    from tests.helpers import oracle_construct, pack_params
    layers = [dict(kind="conv", c_in=1, c_out=1, k=3, s=1, d=1, g=1, padding_mode="circular"),
              dict(kind="conv", c_in=2, c_out=2, k=1, s=1, d=1, g=1, padding_mode="zeros"),
              dict(kind="conv", c_in=1, c_out=4, k=2, s=2, d=1, g=1, padding_mode="circular"),
              dict(kind="conv", c_in=4, c_out=1, k=3, s=1, d=1, g=1, padding_mode="zeros"),
              dict(kind="convT", c_in=1, c_out=4, k=2, s=2, d=1, g=1, padding_mode="circular")]
    plan = cuda_lib.Plan(layers, 0, compute=compute)
    params, mats = pack_params(plan, 12)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    plan.orthogonalize(p, ortho)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    plan.compose(ortho, kf)
    plan.check()
    _, _, o_k = oracle_construct(layers, mats)
    tol = 1e-5 if compute == "f32" else 2e-2
    for l, d in enumerate(layers):
        kg = plan.kernel_f32(kf, l)
        assert rel(kg.cpu().numpy(), o_k[l]) < tol, l
        ci_f, co_f = oracle_layer(d).fwd_channels()
        H = 4
        x = gen.activations((2, H, H, ci_f), (92, l, 0, 0, 1))
        Ho, Wo = plan.out_hw(l, H, H)
        y = torch.empty(2, Ho, Wo, co_f, device="cuda")
        plan.conv_forward(l, kg, torch.from_numpy(x).cuda(), y)
        ref = O.conv2d(nchw(x.astype(np.float64)), o_k[l], s=d["s"], d=1, g=1, mode=d["padding_mode"])
        assert rel(y.cpu().numpy(), nhwc(ref)) < tol, l
        if d["padding_mode"] == "circular" and co_f >= ci_f:   # orthogonal (isometric) layers preserve the norm
            assert abs(np.linalg.norm(y.cpu().numpy()) / np.linalg.norm(x) - 1) < (1e-5 if compute == "f32" else 1e-3)
    plan.check()
