"""f4: SLL x AOC fused down-sampling block on the GPU
against the oracle (App. B.3; readings R28-R30).

* construction: the plan's pre / post AOC layers, the AOL-rescaled SLL kernel,
  and the block's merged kernels C = K (*) K_pre and M = [K_post (*) K_pre |
  -2 K_post (*) K^T] (block convolutions as batched GEMM phases over the emitted
  FP32 kernels) against oracle.sll_block_kernels -- on the oracle's own
  construction (F32 mode) and on the GPU's own pre / post / SLL kernels (both
  modes, which isolates the merge);
* forward: orth_conv_forward on the block (conv C + bias, relu + concat, conv
  M at stride s) against oracle.sll_block_forward with the GPU's kernels
  (elementwise bound) and against the UNFUSED three-layer oracle composition."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from tests.helpers import assert_elementwise, nchw, nhwc, oracle_construct, pack_params, rel, sll_free_kernel

pytestmark = pytest.mark.gpu


def block_layers(c, cs, co, kpre, ks, kpost, s, H):
    return [dict(kind="conv", c_in=c, c_out=c, k=kpre, s=1, d=1, g=1, padding_mode="circular", H=H),
            dict(kind="sll", c_in=c, c_out=cs, k=ks, s=1, d=1, g=1, padding_mode="circular", H=H),
            dict(kind="conv", c_in=c, c_out=co, k=kpost, s=s, d=1, g=1, padding_mode="circular", H=H),
            dict(kind="sll_block", c_in=c, c_out=co, k=1, s=s, d=1, g=1, padding_mode="circular", H=H,
                 pre=0, sll=1, post=2)]


CASES = [(16, 32, 32, 2, 2, 3, 2, 16), (64, 64, 128, 3, 3, 3, 2, 16), (8, 8, 8, 3, 3, 3, 1, 8),
         (32, 16, 64, 2, 3, 4, 2, 12)]


def construct(orth, layers, compute, N):
    plan = orth.Plan(layers, 0, compute=compute, max_batch=N)
    params, mats = pack_params(plan, 23)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    plan.orthogonalize(p, ortho)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
    plan.compose(ortho, kf, kb)
    plan.check()
    return plan, mats, kf, kb


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_sll_block_construction(cuda_lib, case, compute):
    layers = block_layers(*case)
    plan, mats, kf, kb = construct(cuda_lib, layers, compute, 4)
    kf_h = torch.from_numpy(kf.cpu().numpy())
    _, _, o_k = oracle_construct(layers, mats)
    Cg, Mg = [t.numpy() for t in plan.block_kernels(kf_h, 3)]
    Kpre, Ksll, Kpost = [plan.kernel_f32(kf_h, l).numpy().astype(np.float64) for l in range(3)]
    # the SLL layer's kernel: AOL rescale of its free parameters
    assert rel(Ksll, o_k[1]) < (1e-5 if compute == "f32" else 1e-4)
    # the merge alone: the oracle merging the GPU's own three kernels (K_sll already rescaled: rescale is
    # idempotent only up to rounding, so merge with the free W and compare the rescaled factor separately)
    W = sll_free_kernel(layers, 1, mats)
    ref = O.sll_block_kernels(Kpre, Kpost, W)
    assert rel(Cg, ref["C"]) < 1e-4 and rel(Mg, ref["M"]) < 1e-4
    # and end to end against the oracle's construction
    tol = 1e-5 if compute == "f32" else 2e-2
    assert rel(Cg, o_k[3]["C"]) < tol and rel(Mg, o_k[3]["M"]) < tol
    Cb, Mb = [t.float() for t in plan.block_kernels(kb.cpu(), 3)]
    assert np.array_equal(Cb.numpy().transpose(0, 3, 1, 2), gen.bf16_round(Cg.astype(np.float32)))
    assert np.array_equal(Mb.numpy().transpose(0, 3, 1, 2), gen.bf16_round(Mg.astype(np.float32)))


@pytest.mark.parametrize("case", CASES)
def test_sll_block_forward(cuda_lib, case):
    c, cs, co, kpre, ks, kpost, s, H = case
    layers = block_layers(*case)
    N = 4
    plan, mats, kf, kb = construct(cuda_lib, layers, "f32", N)
    kf_h = torch.from_numpy(kf.cpu().numpy())
    Cg, Mg = [t.numpy().astype(np.float64) for t in plan.block_kernels(kf_h, 3)]
    kern = dict(C=Cg, M=Mg, padC=None, padM=None)
    pads = plan.layer_info[3]["pads"]
    pC, pM = pads & 0xFFFF, pads >> 16
    kC, kM = Cg.shape[2], Mg.shape[2]
    kern["padC"] = (pC, kC - 1 - pC, pC, kC - 1 - pC)
    kern["padM"] = (pM, kM - 1 - pM, pM, kM - 1 - pM)
    b = gen.bias(cs, (23, 9, c, cs, 7)) * 10
    x = gen.activations((N, H, H, c), (23, 1, c, co, 6))
    Ho = H // s
    # FP32 I/O: tight, against the fused oracle with the GPU's kernels and the unfused composition
    y = torch.zeros((N, Ho, Ho, co), device="cuda")
    plan.conv_forward(3, plan.block_kernels(kf, 3)[0].reshape(-1), torch.from_numpy(x).cuda(), y,
                      bias=torch.from_numpy(b).cuda())
    plan.check()
    x64 = nchw(x.astype(np.float64))
    ref = O.sll_block_forward(x64, kern, b, s)
    got = y.cpu().numpy()
    assert rel(got, nhwc(ref)) < 1e-5
    Kpre, Kpost = [plan.kernel_f32(kf_h, l).numpy().astype(np.float64) for l in (0, 2)]
    Ksll = plan.kernel_f32(kf_h, 1).numpy().astype(np.float64)
    unf = O.sll_block_unfused(x64, Kpre, Kpost, Ksll, b, s)
    assert rel(got, nhwc(unf)) < 1e-4
    # BF16 I/O through the tensor-core conv kernels where eligible: the BF16 kernels and the BF16 h
    Cb, Mb = [t.float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2) for t in plan.block_kernels(kb, 3)]
    xb = gen.bf16_round(x)
    yb = torch.zeros((N, Ho, Ho, co), device="cuda", dtype=torch.bfloat16)
    plan.conv_forward(3, plan.block_kernels(kb, 3)[0].reshape(-1), torch.from_numpy(xb).cuda().to(torch.bfloat16),
                      yb, bias=torch.from_numpy(b).cuda())
    plan.check()
    xb64 = nchw(xb.astype(np.float64))
    kb_ = dict(kern, C=Cb, M=Mb)
    refb = O.sll_block_forward(xb64, kb_, b, s)
    gotb = yb.float().cpu().numpy()
    assert rel(gotb, nhwc(refb)) < 1e-2
    # elementwise: y's own BF16 rounding + the BF16 rounding of h inside the block (2^-8 of |M_h| |h|)
    h_abs = np.abs(O.conv2d(xb64, Cb, pads=kern["padC"]) + b[None, :, None, None])
    z_abs = np.concatenate([np.abs(xb64), h_abs], axis=1)
    absref = O.conv2d(z_abs, np.abs(Mb), s=s, pads=kern["padM"])
    assert_elementwise(gotb, nhwc(refb), nhwc(absref), 2.0 ** -8, 2.0 ** -7, what=f"block {case} bf16")
