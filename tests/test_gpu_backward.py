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
    # small-kernel SIMT path (E = co ci k^2 <= 4096 per group): grouped, ragged 64-pixel chunks, 7 x 7 zeros
    (8, 8, 3, 2, 1, 2, "zeros", 9, "conv", 3), (3, 24, 7, 2, 1, 1, "zeros", 15, "conv", 3),
    (3, 64, 4, 4, 1, 1, "circular", 224, "conv", 3),
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


# ------------------------------------------------------------------ composition and orthogonalisation VJPs
VJP_LAYERS = [dict(kind=k, c_in=ci, c_out=co, k=kk, s=s, d=1, g=g, padding_mode="circular")
              for (ci, co, kk, s, g, k) in [(16, 16, 3, 1, 1, "conv"), (8, 16, 3, 2, 1, "conv"),
                                            (16, 8, 3, 2, 1, "conv"), (8, 8, 4, 2, 2, "conv"),
                                            (6, 9, 5, 3, 3, "conv"), (3, 64, 4, 4, 1, "conv"),
                                            (12, 20, 2, 1, 1, "conv"), (8, 8, 3, 2, 2, "convT"),
                                            (10, 6, 1, 1, 1, "conv"), (33, 20, 1, 1, 1, "dense"),
                                            (64, 128, 3, 2, 1, "conv")]]


def _grouped(plan, arr, layer_list):
    """per layer: list (groups) of lists (matrices in layer_matrices order) of float64 arrays"""
    out, idx = [], 0
    for l, d in enumerate(layer_list):
        mp = plan.layer_info[l]["mats_per_group"]
        g = 1 if d["kind"] == "dense" else d["g"]
        groups = []
        for _ in range(g):
            ms = []
            for _ in range(mp):
                m = plan.matrices[idx]
                ms.append(arr[m["off"]: m["off"] + m["m"] * m["n"]].reshape(m["m"], m["n"]).astype(np.float64))
                idx += 1
            groups.append(ms)
        out.append(groups)
    return out


@pytest.mark.parametrize("compute,tol", [("f32", 1e-5), ("bf16", 1e-4)])
def test_compose_and_orthogonalize_vjp(cuda_lib, compute, tol):
    """d(ortho) = compose_vjp(dK) against oracle.layer_kernel_vjp on the GPU's own orthogonal matrices, and
    d(params) = orthogonalize_vjp(d(ortho)) against oracle.orthogonalize_vjp (pre-scale constant, R31)."""
    from tests.helpers import pack_params
    plan = cuda_lib.Plan(VJP_LAYERS, 0, compute=compute, vjp=1)
    params, mats = pack_params(plan, 31)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    plan.orthogonalize(p, ortho)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    plan.compose(ortho, kf)
    rng = gen.rng(31, 7)
    dK = torch.from_numpy(rng.standard_normal(plan.kf32_numel).astype(np.float32)).cuda()
    dortho = torch.full_like(p, float("nan"))
    dortho.zero_()
    plan.compose_vjp(ortho, dK, dortho)
    dparams = torch.zeros_like(p)
    plan.orthogonalize_vjp(p, dortho, dparams)
    plan.check()
    o_h, do_h, dp_h, dK_h = (t.cpu().numpy() for t in (ortho, dortho, dparams, dK))
    og, dog = _grouped(plan, o_h, VJP_LAYERS), _grouped(plan, do_h, VJP_LAYERS)
    for l, d in enumerate(VJP_LAYERS):
        OL = oracle_layer(d)
        kshape = plan.kernel_shape(l)
        info = plan.layer_info[l]
        dKl = dK_h[info["kf32_off"]: info["kf32_off"] + info["numel"]].reshape(kshape).astype(np.float64)
        ref = O.layer_kernel_vjp(OL, og[l], dKl)
        for gi in range(len(ref)):
            for j, R in enumerate(ref[gi]):
                if R.size:
                    assert rel(dog[l][gi][j], R) < tol, (l, gi, j, rel(dog[l][gi][j], R))
    # orthogonalize VJP (pre-scale constant: the oracle's own sigma of the same float32 parameters)
    G = [dog_m for groups in dog for ms in groups for dog_m in ms]
    refp = O.orthogonalize_vjp([A.astype(np.float64) for A in mats], G, T=12)
    for i, m in enumerate(plan.matrices):
        if m["m"] * m["n"] == 0:
            continue
        got = dp_h[m["off"]: m["off"] + m["m"] * m["n"]].reshape(m["m"], m["n"])
        assert rel(got, refp[i]) < tol, (i, m, rel(got, refp[i]))


def test_whole_path_gradient_cfg1(cuda_lib):
    """End to end on config 1: L = <G, conv(x, K(params))>; wgrad -> compose VJP -> orthogonalize VJP on the
    GPU (FP32) against the oracle chain of VJPs, and against a central finite difference of L through the
    ORACLE forward (pre-scale held at the oracle's sigma, R31)."""
    from synth import configs
    from tests.helpers import nhwc, pack_params
    layers = configs.cfg1()
    plan = cuda_lib.Plan(layers, 0, vjp=1)
    params, mats = pack_params(plan, 1)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    plan.orthogonalize(p, ortho)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    plan.compose(ortho, kf)
    x = gen.activations((2, 8, 8, 16), (1, 0, 0, 0, gen.ROLE_ID["x"]))
    Gy = gen.activations((2, 8, 8, 16), (1, 0, 0, 1, gen.ROLE_ID["x"]))
    dK = torch.zeros(plan.kf32_numel, device="cuda")
    plan.conv_wgrad(0, torch.from_numpy(x).cuda(), torch.from_numpy(Gy).cuda(),
                    plan.kernel_f32(dK, 0))
    dortho = torch.zeros_like(p)
    plan.compose_vjp(ortho, dK, dortho)
    dparams = torch.zeros_like(p)
    plan.orthogonalize_vjp(p, dortho, dparams)
    plan.check()
    OL = oracle_layer(layers[0])
    x64, G64 = nchw(x.astype(np.float64)), nchw(Gy.astype(np.float64))
    o_ortho, _ = O.orthogonalize([A.astype(np.float64) for A in mats], T=12)
    K = O.layer_kernel(OL, [o_ortho])
    dK_o = O.conv2d_wgrad(x64, G64, K.shape)
    dmats = O.layer_kernel_vjp(OL, [o_ortho], dK_o)[0]
    dW_o = O.orthogonalize_vjp([A.astype(np.float64) for A in mats], dmats, T=12)
    dp_h = dparams.cpu().numpy()
    sig = [O.prescale_power(A.astype(np.float64), 3, np.ones(A.shape[1]) / np.sqrt(A.shape[1]))[1] for A in mats]
    rng = gen.rng(1, 99)
    for i, m in enumerate(plan.matrices):
        got = dp_h[m["off"]: m["off"] + m["m"] * m["n"]].reshape(m["m"], m["n"])
        assert rel(got, dW_o[i]) < 1e-4, (i, rel(got, dW_o[i]))
        D = rng.standard_normal(mats[i].shape)
        eps = 1e-5

        def loss(Ai):
            ms = [A.astype(np.float64) for A in mats]
            ms[i] = Ai
            o = [O.bjorck(A / sg, 12) for A, sg in zip(ms, sig)]
            return float((G64 * O.conv2d(x64, O.layer_kernel(OL, [o]))).sum())
        A0 = mats[i].astype(np.float64)
        fd = (loss(A0 + eps * D) - loss(A0 - eps * D)) / (2 * eps)
        assert abs(fd - float((dW_o[i] * D).sum())) < 1e-5 * max(1.0, abs(fd))
        assert abs(fd - float((got * D).sum())) < 1e-3 * max(1.0, abs(fd))
