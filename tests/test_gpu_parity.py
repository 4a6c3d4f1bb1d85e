"""GPU parity: the CUDA path through the C ABI against the float64 oracle on
the same seeded inputs.  Tolerances (north star, reading R18): per tensor
|gpu - oracle|_F / |oracle|_F <= 1e-5 for the FP32 path, <= 2e-2 for BF16;
orthogonality max|sigma - 1| <= 1e-3 of the GPU's FP32 kernels."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import configs, gen
from tests.helpers import (BF16_ELEM, F32_ELEM, assert_elementwise, nchw, nhwc, oracle_construct, oracle_layer,
                           pack_cache, pack_params, rel)

pytestmark = pytest.mark.gpu

TOL32, TOL16 = 1e-5, 2e-2


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def gpu_construct(orth, layers, cfg_id, stress=False, with_cache=False, **opts):
    plan = orth.Plan(layers, 0, **opts)
    params, mats = pack_params(plan, cfg_id, stress)
    p = dev(params)
    ortho = torch.zeros_like(p)
    res = torch.full((plan.n_matrices,), -1.0, device="cuda")
    cache, vs = (None, None)
    if with_cache:
        cbuf, vs = pack_cache(plan, cfg_id)
        cache = dev(cbuf)
    plan.orthogonalize(p, ortho, cache, res)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
    plan.compose(ortho, kf, kb)
    plan.check()
    return plan, mats, vs, ortho, res, cache, kf, kb


def unpack(plan, buf, i):
    m = plan.matrices[i]
    return buf[m["off"]: m["off"] + m["m"] * m["n"]].reshape(m["m"], m["n"])


# ------------------------------------------------------------------ construction
@pytest.mark.parametrize("cfg_id,layers", [(1, configs.cfg1()),
                                           (11, [dict(kind=k, c_in=ci, c_out=co, k=kk, s=s, d=d, g=g,
                                                      padding_mode="circular")
                                                 for (ci, co, kk, s, d, g, k) in [
                                                     (4, 8, 3, 2, 1, 1, "conv"), (8, 4, 3, 2, 1, 1, "conv"),
                                                     (1, 8, 3, 2, 1, 1, "conv"), (4, 16, 2, 2, 1, 1, "conv"),
                                                     (8, 8, 4, 2, 1, 1, "conv"), (1, 1, 3, 1, 1, 1, "conv"),
                                                     (8, 16, 3, 2, 1, 2, "conv"), (8, 8, 3, 1, 2, 2, "convT"),
                                                     (4, 8, 3, 2, 1, 2, "convT"), (6, 9, 5, 3, 2, 3, "conv"),
                                                     (3, 64, 4, 4, 1, 1, "conv"), (96, 80, 3, 1, 1, 1, "conv"),
                                                     (70, 70, 1, 1, 1, 1, "dense"), (33, 130, 1, 1, 1, 1, "dense")]])])
@pytest.mark.parametrize("with_cache", [False, True])
def test_construction_parity_fp32(cuda_lib, cfg_id, layers, with_cache):
    plan, mats, vs, ortho, res, cache, kf, kb = gpu_construct(cuda_lib, layers, cfg_id, with_cache=with_cache)
    o_ortho, o_v, o_k = oracle_construct(layers, mats, v=vs)
    ortho_h, res_h, kf_h = ortho.cpu().numpy(), res.cpu().numpy(), kf.cpu().numpy()
    kb_h = kb.float().cpu().numpy()
    for i, X in enumerate(o_ortho):
        if X.size == 0:
            continue
        assert rel(unpack(plan, ortho_h, i), X) < TOL32, (i, plan.matrices[i])
        assert abs(res_h[i] - O.ns_residual(X)) < 1e-4
        if with_cache:
            m = plan.matrices[i]
            vg = cache.cpu().numpy()[m["cache_off"]: m["cache_off"] + m["n"]]
            assert rel(vg, o_v[i]) < 1e-4
    for l, K in enumerate(o_k):
        kg = plan.kernel_f32(torch.from_numpy(kf_h), l).numpy()
        assert kg.shape == K.shape
        assert rel(kg, K) < TOL32, l
        kbg = plan.kernel_bf16(torch.from_numpy(kb_h), l).numpy()
        if K.ndim == 4:
            kbg = np.transpose(kbg, (0, 3, 1, 2))
        assert np.array_equal(kbg, gen.bf16_round(kg.astype(np.float32)))   # emit is an RNE cast of the FP32 kernel


def test_gpu_kernels_orthogonal_toeplitz(cuda_lib):
    # P:462 explicit Toeplitz SVD on 8x8 inputs, applied to the GPU's FP32 kernels
    layers = [dict(kind="conv", c_in=ci, c_out=co, k=k, s=s, d=1, g=g, padding_mode="circular")
              for (ci, co, k, s, g) in [(16, 16, 3, 1, 1), (4, 8, 3, 2, 1), (8, 4, 3, 2, 1), (4, 32, 3, 2, 1),
                                        (8, 8, 4, 2, 2), (4, 16, 2, 2, 1)]]
    plan, mats, _, _, _, _, kf, _ = gpu_construct(cuda_lib, layers, 12)
    kf_h = torch.from_numpy(kf.cpu().numpy())
    for l, d in enumerate(layers):
        K = plan.kernel_f32(kf_h, l).numpy().astype(np.float64)
        OL = oracle_layer(d)
        T = O.toeplitz(lambda x: O.conv2d(x, K, s=OL.s, d=OL.d, g=OL.g), (d["c_in"], 8, 8))
        sv = np.linalg.svd(T, compute_uv=False)[: min(T.shape)]
        assert np.abs(sv - 1).max() < 1e-3, (l, sv.min(), sv.max())


def test_construction_cfg2_full(cuda_lib):
    layers = configs.cfg2()
    plan, mats, _, ortho, res, _, kf, _ = gpu_construct(cuda_lib, layers, 2)
    o_ortho, _, o_k = oracle_construct(layers, mats)
    ortho_h, kf_h = ortho.cpu().numpy(), torch.from_numpy(kf.cpu().numpy())
    for i, X in enumerate(o_ortho):
        assert rel(unpack(plan, ortho_h, i), X) < TOL32
    for l, K in enumerate(o_k):
        assert rel(plan.kernel_f32(kf_h, l).numpy(), K) < TOL32
    assert float(res.max()) < 1e-3


def test_frobenius_and_stress(cuda_lib):
    layers = [dict(kind="conv", c_in=16, c_out=16, k=3, s=1, d=1, g=1, padding_mode="circular"),
              dict(kind="dense", c_in=48, c_out=20, k=1, s=1, d=1, g=1, padding_mode="circular")]
    plan, mats, _, ortho, res, _, kf, _ = gpu_construct(cuda_lib, layers, 13, stress=True, prescale="frobenius",
                                                        ns_iters=40)
    o_ortho, _, o_k = oracle_construct(layers, mats, T=40, prescale="frobenius")
    ortho_h = ortho.cpu().numpy()
    for i, X in enumerate(o_ortho):
        assert rel(unpack(plan, ortho_h, i), X) < TOL32
    assert float(res.max()) < 1e-4


def test_determinism(cuda_lib):
    layers = configs.cfg2()[:5]
    a = gpu_construct(cuda_lib, layers, 2)
    b = gpu_construct(cuda_lib, layers, 2)
    assert torch.equal(a[3], b[3]) and torch.equal(a[6], b[6]) and torch.equal(a[7], b[7])


def test_device_status_zero_and_nonconvergence(cuda_lib):
    orth = cuda_lib
    layers = [dict(kind="dense", c_in=2, c_out=2, k=1, s=1, d=1, g=1, padding_mode="circular")]
    plan = orth.Plan(layers, 0, power_iters=1)
    p = torch.zeros(plan.params_numel, device="cuda")
    plan.orthogonalize(p, torch.zeros_like(p))
    with pytest.raises(orth.OrthError) as ei:
        plan.check()
    assert ei.value.status == orth.ZERO_NORM
    # sigma underestimated by a start vector orthogonal to the top singular vector -> divergence (R20)
    p[0] = 100.0
    p[3] = 1e-3
    cache = torch.zeros(plan.cache_numel, device="cuda")
    cache[1] = 1.0
    res = torch.zeros(1, device="cuda")
    plan.orthogonalize(p, torch.zeros_like(p), cache, res)
    with pytest.raises(orth.OrthError) as ei:
        plan.check()
    assert ei.value.status == orth.NOT_CONVERGED
    plan.check()                                              # cleared


@pytest.mark.parametrize("mode", ["f32", "bf16"])
def test_not_converged_without_residual_out(cuda_lib, mode):
    """S:125 non-convergence is reported whether or not residual_out is requested: the
    last iteration's own Gram gives r = |I - X_{T-1}^T X_{T-1}|_F and the bound 3/4 r^2 + 1/4 r^3 on the
    result's residual is checked against ns_tol.  Gaussian (stress) matrices at T = 3 are far from
    converged (R21); at T = 40 with Frobenius pre-scaling they converge; ns_tol <= 0 keeps only the
    non-finite check."""
    orth = cuda_lib
    layers = [dict(kind="dense", c_in=96, c_out=96, k=1, s=1, d=1, g=1, padding_mode="circular"),
              dict(kind="conv", c_in=16, c_out=16, k=3, s=1, d=1, g=1, padding_mode="circular")]
    for T, tol, expect in [(3, 1e-3, orth.NOT_CONVERGED), (40, 1e-3, orth.OK), (3, 0.0, orth.OK)]:
        plan = orth.Plan(layers, 0, compute=mode, ns_iters=T, prescale="frobenius", ns_tol=tol)
        params, _ = pack_params(plan, 16, stress=True)
        p = dev(params)
        plan.orthogonalize(p, torch.zeros_like(p))      # residual_out = NULL
        if expect == orth.OK:
            plan.check()
        else:
            with pytest.raises(orth.OrthError) as ei:
                plan.check()
            assert ei.value.status == expect
            plan.check()                                # the status word is cleared by the check


# ------------------------------------------------------------------ conv apply
CONV_CASES = [  # (ci, co, k, s, d, g, mode, H, kind)
    (16, 16, 3, 1, 1, 1, "circular", 8, "conv"), (3, 64, 3, 1, 1, 1, "circular", 32, "conv"),
    (64, 128, 3, 2, 1, 1, "circular", 16, "conv"), (24, 40, 3, 2, 1, 1, "zeros", 9, "conv"),
    (32, 32, 3, 1, 2, 4, "circular", 12, "conv"), (12, 18, 5, 3, 2, 3, "zeros", 11, "conv"),
    (3, 64, 4, 4, 1, 1, "circular", 16, "conv"), (20, 20, 2, 1, 1, 1, "zeros", 7, "conv"),
    (96, 80, 3, 2, 1, 1, "circular", 10, "convT"), (32, 32, 3, 1, 2, 8, "circular", 9, "convT"),
    (17, 33, 3, 2, 1, 1, "zeros", 7, "convT"), (130, 70, 1, 1, 1, 1, "zeros", 5, "conv"),
    # tcgen05-eligible shapes (co_g % 64 == 0, ci_g % 8 == 0) incl. ragged pixel tiles and channel tails
    (64, 64, 3, 1, 1, 1, "circular", 10, "conv"), (64, 64, 3, 1, 1, 1, "zeros", 9, "conv"),
    (128, 256, 3, 2, 1, 1, "circular", 8, "conv"), (256, 512, 3, 2, 1, 1, "zeros", 7, "conv"),
    (64, 64, 3, 1, 2, 1, "circular", 12, "conv"), (128, 128, 3, 1, 1, 2, "circular", 8, "conv"),
    (40, 64, 3, 1, 1, 1, "circular", 6, "conv"), (72, 128, 5, 2, 1, 1, "zeros", 9, "conv"),
    (512, 512, 3, 1, 1, 1, "circular", 4, "conv"), (64, 128, 3, 2, 3, 1, "circular", 12, "conv"),
    (8, 32, 2, 2, 1, 2, "zeros", 9, "conv"), (3, 64, 3, 1, 1, 1, "zeros", 13, "conv"),
    # tensor-core adjoint (polyphase tiles) and 32-wide output tiles (grouped layers)
    (64, 64, 3, 2, 1, 1, "circular", 8, "convT"), (128, 64, 3, 2, 1, 1, "zeros", 9, "conv"),
    (64, 64, 3, 1, 2, 2, "circular", 12, "convT"), (256, 256, 3, 1, 1, 8, "circular", 8, "conv"),
    (64, 128, 4, 2, 1, 1, "zeros", 10, "convT"), (96, 96, 5, 3, 2, 3, "circular", 12, "conv"),
    (64, 128, 3, 2, 1, 1, "zeros", 9, "conv"), (1024, 1024, 3, 1, 2, 32, "circular", 6, "convT"),
    # stride-1 shifted-copy A-reuse path (TH x Wo tiles >= 96 rows; ragged Wo: descriptor starts inside a swizzle atom)
    (64, 64, 3, 1, 1, 1, "zeros", 16, "conv"), (128, 128, 3, 1, 1, 1, "circular", 16, "conv"),
    (64, 128, 3, 1, 1, 1, "circular", 32, "conv"), (32, 32, 3, 1, 1, 2, "circular", 16, "conv"),
    (256, 256, 3, 1, 1, 1, "zeros", 12, "conv"), (64, 64, 5, 1, 1, 1, "circular", 20, "conv"),
    (64, 64, 3, 1, 3, 1, "zeros", 14, "conv"), (192, 64, 3, 1, 1, 1, "circular", 11, "conv"),
    # TMA-window path (conv_pad.cu: co_g <= 64, Wo >= 16): resident / streamed weights, channel tails
    (64, 64, 3, 1, 1, 1, "circular", 24, "conv"), (64, 64, 5, 1, 2, 1, "zeros", 20, "conv"),
    (48, 64, 3, 1, 1, 1, "circular", 16, "conv"), (128, 64, 3, 1, 1, 1, "circular", 16, "conv"),
    (64, 32, 3, 1, 1, 1, "zeros", 33, "conv"),
    # stride-1 adjoints on the TMA-window path (tap-flipped forward form), incl. packed groups
    (64, 64, 3, 1, 1, 1, "circular", 24, "convT"), (64, 64, 3, 1, 2, 1, "zeros", 20, "convT"),
    (64, 64, 3, 1, 2, 2, "circular", 20, "convT"), (1024, 1024, 3, 1, 2, 32, "circular", 16, "convT"),
    (128, 64, 5, 1, 1, 1, "zeros", 17, "convT"),
    # stacked-window path (conv_stack.cu: >= 128 output channels, several small images per tile)
    (128, 256, 3, 1, 2, 1, "circular", 12, "conv"), (256, 128, 5, 1, 1, 1, "zeros", 9, "conv"),
    (128, 128, 3, 1, 1, 1, "circular", 7, "conv"), (256, 256, 3, 1, 1, 2, "circular", 8, "conv"),
    (128, 128, 3, 1, 1, 1, "zeros", 30, "conv"), (512, 512, 3, 1, 1, 1, "circular", 5, "convT"),
    (1024, 1024, 3, 1, 2, 1, "circular", 8, "conv"), (96, 128, 3, 1, 1, 1, "circular", 6, "conv"),
    # large kernels on the gather path (8 <= k <= 13: the SOC explicit exponential's k_eff = 13; shallower
    # rings around the 86.5 KB pixel table), every N-tile width, strided and adjoint
    (64, 64, 13, 1, 1, 1, "circular", 16, "conv"), (128, 128, 9, 1, 1, 1, "zeros", 12, "conv"),
    (64, 128, 11, 2, 1, 1, "zeros", 15, "conv"), (256, 256, 13, 1, 1, 1, "circular", 13, "conv"),
    (64, 64, 9, 2, 1, 1, "circular", 10, "convT"), (32, 32, 13, 1, 1, 1, "circular", 14, "conv"),
]


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("io", ["f32", "bf16"])
def test_conv_forward_and_transpose(cuda_lib, case, io, max_batch=None):
    ci, co, k, s, d, g, mode, H, kind = case
    layer = dict(kind=kind, c_in=ci, c_out=co, k=k, s=s, d=d, g=g, padding_mode=mode)
    OL = oracle_layer(layer)
    ci_f, co_f = OL.fwd_channels()
    rng = gen.rng(77, ci, co, k, s)
    K = (rng.standard_normal((co_f, ci_f // g, k, k)) / np.sqrt(ci_f // g * k * k)).astype(np.float32)
    N = 3
    Hb = H * s if (kind == "convT" and mode == "circular") else H
    x = gen.activations((N, Hb, Hb + 1 if mode == "zeros" else Hb, ci_f), (77, 1, ci, co, 6))
    bias = gen.bias(co_f, (77, 2, ci, co, 7))
    if io == "bf16":
        K, x = gen.bf16_round(K), gen.bf16_round(x)
        kdev = dev(np.transpose(K, (0, 2, 3, 1)), torch.bfloat16)
        xdev, tdt, tol = dev(x, torch.bfloat16), torch.bfloat16, TOL16
    else:
        kdev, xdev, tdt, tol = dev(K), dev(x), torch.float32, TOL32
    Hh, Ww = x.shape[1], x.shape[2]
    # the declared grid and batch size the layer's conv scratch at create (split-K, padded-copy kernels)
    plan = cuda_lib.Plan([dict(layer, grid=(Hh, Ww))], 0, max_batch=N if max_batch is None else max_batch)
    Ho, Wo = plan.out_hw(0, Hh, Ww)
    y = torch.zeros((N, Ho, Wo, co_f), device="cuda", dtype=tdt)
    plan.conv_forward(0, kdev, xdev, y, bias=dev(bias))
    K64, x64 = K.astype(np.float64), nchw(x.astype(np.float64))
    ref = O.conv2d(x64, K64, s=s, d=d, g=g, mode=mode) + bias[None, :, None, None]
    absref = O.conv2d(np.abs(x64), np.abs(K64), s=s, d=d, g=g, mode=mode) + np.abs(bias)[None, :, None, None]
    elem = BF16_ELEM if io == "bf16" else F32_ELEM
    got = y.float().cpu().numpy()
    assert rel(got, nhwc(ref)) < (1e-2 if io == "bf16" else tol)
    assert_elementwise(got, nhwc(ref), nhwc(absref), *elem, what=f"forward {case} {io}")
    # adjoint
    yr = gen.activations((N, Ho, Wo, co_f), (77, 3, ci, co, 6))
    if io == "bf16":
        yr = gen.bf16_round(yr)
    xb = torch.zeros((N, Hh, Ww, ci_f), device="cuda", dtype=tdt)
    plan.conv_transpose(0, kdev, dev(yr, tdt), xb)
    yr64 = nchw(yr.astype(np.float64))
    refT = O.conv_transpose2d(yr64, K64, Hh, Ww, s=s, d=d, g=g, mode=mode)
    absT = O.conv_transpose2d(np.abs(yr64), np.abs(K64), Hh, Ww, s=s, d=d, g=g, mode=mode)
    gotT = xb.float().cpu().numpy()
    assert rel(gotT, nhwc(refT)) < (1e-2 if io == "bf16" else tol)
    assert_elementwise(gotT, nhwc(refT), nhwc(absT), *elem, what=f"adjoint {case} {io}")
    plan.check()


# Split-K of the gather conv (two half-K items per 128 x 256 tile, FP32 partial + flag in the layer's
# scratch): deep layers with few 256-wide tiles, in both directions; each case also runs with the
# scratch withheld (max_batch = 0: no split) and both results must satisfy the same elementwise bound.
SPLITK_CASES = [(512, 512, 3, 1, 1, 1, "circular", 4, "conv"), (1024, 1024, 3, 1, 1, 1, "zeros", 4, "conv"),
                (512, 512, 3, 2, 1, 1, "circular", 8, "conv"), (1024, 1024, 3, 1, 2, 1, "circular", 6, "convT"),
                (768, 512, 5, 2, 1, 1, "zeros", 7, "conv")]


@pytest.mark.parametrize("case", SPLITK_CASES)
def test_conv_splitk_path(cuda_lib, case):
    ci, co, k, s, d, g, mode, H, kind = case
    layer = dict(kind=kind, c_in=ci, c_out=co, k=k, s=s, d=d, g=g, padding_mode=mode)
    Hb = H * s if (kind == "convT" and mode == "circular") else H
    plan = cuda_lib.Plan([dict(layer, grid=(Hb, Hb + 1 if mode == "zeros" else Hb))], 0, max_batch=3)
    assert plan.layer_info[0]["scratch"] >= 128 * 256 * 4, "case does not reach split-K"
    test_conv_forward_and_transpose(cuda_lib, case, "bf16")               # with split-K
    test_conv_forward_and_transpose(cuda_lib, case, "bf16", max_batch=0)  # without


@pytest.mark.parametrize("case", [(128, 128, 3, 1, 1, 1, "circular", 16, "conv"), (128, 256, 3, 2, 1, 1, "zeros", 9, "conv"),
                                  (256, 256, 3, 1, 2, 1, "circular", 8, "convT")])
def test_conv_pair_path(cuda_lib, case):
    """The opt-in 2-SM pair (cta_group::2) conv kernel, in a subprocess (the switch is read once); built only
    with ORTH_EXPERIMENTAL=1."""
    if not cuda_lib.experimental():
        pytest.skip("experimental kernels not built (ORTH_EXPERIMENTAL=1)")
    import os
    import subprocess
    import sys
    code = (f"import sys; sys.path.insert(0, {os.getcwd()!r}); import tests.test_gpu_parity as t; "
            f"import paper_2601_13776_b200 as orth; t.test_conv_forward_and_transpose(orth, {case!r}, 'bf16')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "ORTH_CONV_PAIR": "1"},
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


ROW_CASES = [(64, 64, 3, 1, 1, 1, "circular", 10, "conv"), (64, 64, 3, 1, 1, 1, "zeros", 9, "conv"),
             (64, 64, 3, 1, 2, 1, "circular", 12, "conv"), (64, 64, 2, 1, 1, 1, "circular", 9, "conv"),
             (192, 64, 3, 1, 1, 1, "circular", 11, "conv"), (64, 64, 3, 1, 1, 1, "circular", 24, "convT"),
             (64, 64, 3, 1, 1, 1, "circular", 24, "conv")]


@pytest.mark.parametrize("switch", ["ORTH_CONV_ROW", "ORTH_CONV_NO_SWAP", "ORTH_CONV_NO_BRES"])
def test_conv_64_channel_forms(switch):
    """The 64-output-channel layers' alternative forms, in a subprocess (the switches are read once): the
    opt-in kernel-row MMAs (ORTH_CONV_ROW=1), the one-chain-per-tap form with M = 128 pixels
    (ORTH_CONV_NO_SWAP=1, two MMA issuers on a resident weight set) and the default swapped form with
    streamed instead of resident weights (ORTH_CONV_NO_BRES=1, one issuer); forward and adjoint, BF16."""
    import os
    import subprocess
    import sys
    code = (f"import sys; sys.path.insert(0, {os.getcwd()!r}); import tests.test_gpu_parity as t; "
            f"import paper_2601_13776_b200 as orth\n"
            f"for c in {ROW_CASES!r}: t.test_conv_forward_and_transpose(orth, c, 'bf16')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, switch: "1"}, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


STACK_CASES = [(128, 256, 3, 1, 2, 1, "circular", 12, "conv"), (256, 128, 5, 1, 1, 1, "zeros", 9, "conv"),
               (128, 128, 3, 1, 1, 1, "circular", 7, "conv"), (256, 256, 3, 1, 1, 2, "circular", 8, "conv"),
               (128, 128, 3, 1, 1, 1, "zeros", 30, "conv"), (512, 512, 3, 1, 1, 1, "circular", 5, "convT"),
               (96, 128, 3, 1, 1, 1, "circular", 6, "conv"), (512, 512, 3, 1, 1, 1, "circular", 4, "conv")]


def test_conv_tma_path(cuda_lib):
    """The opt-in TMA implicit-GEMM kernel (conv_tma.cu, ORTH_CONV_TMA=1: padded copy + one 4-D box per
    tap) on stride-1 >= 128-channel cases, forward and adjoint, BF16, in a subprocess; built only with
    ORTH_EXPERIMENTAL=1."""
    if not cuda_lib.experimental():
        pytest.skip("experimental kernels not built (ORTH_EXPERIMENTAL=1)")
    import os
    import subprocess
    import sys
    code = (f"import sys; sys.path.insert(0, {os.getcwd()!r}); import tests.test_gpu_parity as t; "
            f"import paper_2601_13776_b200 as orth\n"
            f"for c in {STACK_CASES!r}: t.test_conv_forward_and_transpose(orth, c, 'bf16')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "ORTH_CONV_TMA": "1"},
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_conv_stack_path():
    """The opt-in stacked-window kernel (conv_stack.cu, ORTH_CONV_STACK=1) on the same parity cases, in a
    subprocess (the switch is read once); forward and adjoint, BF16."""
    import os
    import subprocess
    import sys
    code = (f"import sys; sys.path.insert(0, {os.getcwd()!r}); import tests.test_gpu_parity as t; "
            f"import paper_2601_13776_b200 as orth\n"
            f"for c in {STACK_CASES!r}: t.test_conv_forward_and_transpose(orth, c, 'bf16')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "ORTH_CONV_STACK": "1"},
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_conv_rejections(cuda_lib):
    orth = cuda_lib
    plan = orth.Plan([dict(kind="conv", c_in=4, c_out=4, k=3, s=2, d=1, g=1, padding_mode="circular"),
                      dict(kind="dense", c_in=4, c_out=4, k=1, s=1, d=1, g=1, padding_mode="circular")], 0)
    K = torch.zeros(4 * 4 * 9, device="cuda")
    x = torch.zeros((1, 9, 9, 4), device="cuda")
    y = torch.zeros((1, 5, 5, 4), device="cuda")
    with pytest.raises(orth.OrthError) as ei:
        plan.conv_forward(0, K, x, y)
    assert ei.value.status == orth.SHAPE_MISMATCH          # circular with s not dividing H (R11)
    with pytest.raises(orth.OrthError) as ei:
        plan.conv_forward(1, K, x, y)
    assert ei.value.status == orth.UNSUPPORTED_CONFIG


# ------------------------------------------------------------------ whole path, cfg1 and cfg2
def test_whole_path_cfg1_norm_preserving(cuda_lib):
    layers = configs.cfg1()
    plan, mats, _, _, _, _, kf, kb = gpu_construct(cuda_lib, layers, 1)
    _, _, o_k = oracle_construct(layers, mats)
    x = gen.activations((2, 8, 8, 16), (1, 0, 0, 0, gen.ROLE_ID["x"]))
    y = torch.zeros((2, 8, 8, 16), device="cuda")
    plan.conv_forward(0, plan.kernel_f32(kf, 0), dev(x), y)
    ref = nhwc(O.conv2d(nchw(x.astype(np.float64)), o_k[0]))
    yh = y.cpu().numpy()
    assert rel(yh, ref) < TOL32
    nx = np.sqrt((x.astype(np.float64) ** 2).sum(axis=(1, 2, 3)))
    ny = np.sqrt((yh.astype(np.float64) ** 2).sum(axis=(1, 2, 3)))
    assert np.abs(ny / nx - 1).max() < 1e-5


def test_whole_path_cfg2_bf16_chain_sampled(cuda_lib):
    """Full-size cfg2 step as bench.py runs it (batch 256, bf16 chain); the
    oracle chains its own kernels on a 2-image sample."""
    layers = configs.cfg2()
    plan, mats, _, _, _, _, kf, kb = gpu_construct(cuda_lib, layers, 2, max_batch=256)
    _, _, o_k = oracle_construct(layers, mats)
    N = 256
    x = gen.bf16_round(gen.activations((N, 32, 32, 3), (2, 0, 0, 0, gen.ROLE_ID["x"])))
    cur = dev(x, torch.bfloat16)
    H = 32
    outs = []
    for l, d in enumerate(layers):
        Ho, _ = plan.out_hw(l, H, H)
        y = torch.empty((N, Ho, Ho, d["c_out"]), device="cuda", dtype=torch.bfloat16)
        plan.conv_forward(l, plan.kernel_bf16(kb, l), cur, y)
        outs.append(y)
        cur, H = y, Ho
    plan.check()
    sample = [0, 255]
    ref = nchw(x[sample].astype(np.float64))
    xin = ref
    for l, d in enumerate(layers):
        OL = oracle_layer(d)
        ref = O.conv2d(ref, o_k[l], s=OL.s, d=OL.d, g=OL.g)
        got = outs[l][sample].float().cpu().numpy()
        assert rel(got, nhwc(ref)) < TOL16, l
        # elementwise: the oracle conv with the GPU's own BF16 kernel on the GPU's own input of this layer
        kg = plan.kernel_bf16(kb, l).float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2)
        r1 = O.conv2d(xin, kg, s=OL.s, d=OL.d, g=OL.g)
        a1 = O.conv2d(np.abs(xin), np.abs(kg), s=OL.s, d=OL.d, g=OL.g)
        assert_elementwise(got, nhwc(r1), nhwc(a1), *BF16_ELEM, what=f"cfg2 layer {l}")
        xin = nchw(got)
    # property at any size: circular isometries / co-isometries never increase the norm
    xn = torch.linalg.vector_norm(dev(x).reshape(N, -1), dim=1)
    yn = torch.linalg.vector_norm(outs[-1].float().reshape(N, -1), dim=1)
    assert bool((yn <= xn * 1.02).all())


# ------------------------------------------------------------------ tensor-core construction modes
TC_LAYERS = [dict(kind=k, c_in=ci, c_out=co, k=kk, s=s, d=d, g=g, padding_mode="circular")
             for (ci, co, kk, s, d, g, k) in [
                 (16, 16, 3, 1, 1, 1, "conv"), (4, 8, 3, 2, 1, 1, "conv"), (8, 16, 3, 2, 1, 2, "conv"),
                 (6, 9, 5, 3, 2, 3, "conv"), (3, 64, 4, 4, 1, 1, "conv"), (96, 80, 3, 1, 1, 1, "conv"),
                 (4, 8, 3, 2, 1, 2, "convT"), (70, 70, 1, 1, 1, 1, "dense"), (33, 130, 1, 1, 1, 1, "dense"),
                 (200, 136, 1, 1, 1, 1, "dense")]]


# bf16x3: every product through the 3-pass hi/lo split (~2^-16); measured ~2e-5 on chained BCOP kernels, so 1e-4
@pytest.mark.parametrize("mode,tol", [("bf16", TOL16), ("bf16x3", 1e-4)])
@pytest.mark.parametrize("which", ["small", "cfg2"])
def test_construction_parity_tensor_cores(cuda_lib, mode, tol, which):
    layers = TC_LAYERS if which == "small" else configs.cfg2()
    cfg_id = 14 if which == "small" else 2
    plan, mats, _, ortho, res, _, kf, kb = gpu_construct(cuda_lib, layers, cfg_id, compute=mode)
    o_ortho, _, o_k = oracle_construct(layers, mats)
    ortho_h, kf_h = ortho.cpu().numpy(), torch.from_numpy(kf.cpu().numpy())
    worst = 0.0
    for i, X in enumerate(o_ortho):
        if X.size == 0:
            continue
        e = rel(unpack(plan, ortho_h, i), X)
        worst = max(worst, e)
        assert e < tol, (i, plan.matrices[i], e)
    for l, K in enumerate(o_k):
        assert rel(plan.kernel_f32(kf_h, l).numpy(), K) < tol, l
    # orthogonality of the result (north star: max|sigma - 1| <= 1e-3); |I - X^T X|_F bounds it
    assert float(res.max()) < 1e-3
    print(f"{mode} {which}: worst matrix rel err {worst:.2e}, max residual {float(res.max()):.2e}")


def test_tensor_core_kernels_orthogonal_toeplitz(cuda_lib):
    layers = [dict(kind="conv", c_in=ci, c_out=co, k=k, s=s, d=1, g=g, padding_mode="circular")
              for (ci, co, k, s, g) in [(16, 16, 3, 1, 1), (4, 8, 3, 2, 1), (8, 8, 4, 2, 2)]]
    plan, _, _, _, _, _, kf, _ = gpu_construct(cuda_lib, layers, 15, compute="bf16")
    kf_h = torch.from_numpy(kf.cpu().numpy())
    for l, d in enumerate(layers):
        K = plan.kernel_f32(kf_h, l).numpy().astype(np.float64)
        OL = oracle_layer(d)
        T = O.toeplitz(lambda x: O.conv2d(x, K, s=OL.s, d=OL.d, g=OL.g), (d["c_in"], 8, 8))
        sv = np.linalg.svd(T, compute_uv=False)[: min(T.shape)]
        assert np.abs(sv - 1).max() < 1e-3, (l, sv.min(), sv.max())
