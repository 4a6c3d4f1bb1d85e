"""Full-size parity for the BASELINE.json configurations that are not the bench
line (cfg3 ImageNet AOC-ResNet34 shape, cfg4 1024-channel paths, cfg5 dense
sweep), in the launch configuration bench.py uses (BF16 construction, BF16
activations, batch 256).  The oracle computes what it can one by one:

* construction: every matrix and every composed kernel of cfg3 / cfg4 against
  the float64 oracle (TOL16), orthogonality residual <= 1e-3 (north star);
* forward: per layer, the GPU output of sampled images against the oracle conv
  applied to the SAME GPU input (so errors do not compound with depth), with
  the oracle's own kernels;
* cfg5: all 64 matrices' residuals at n = 4096 and 8192 (a property that holds
  at any size) and one n = 2048 matrix against the oracle.

Reading R18: |gpu - oracle|_F / |oracle|_F per tensor."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import configs, gen
from tests.helpers import BF16_ELEM, assert_elementwise, nchw, nhwc, oracle_construct, oracle_layer, pack_params, rel

pytestmark = pytest.mark.gpu

TOL16 = 2e-2


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def construct_bf16(orth, layers, cfg_id, max_batch=0):
    plan = orth.Plan(layers, 0, compute="bf16", max_batch=max_batch)
    params, mats = pack_params(plan, cfg_id)
    p = dev(params)
    ortho = torch.zeros_like(p)
    res = torch.full((plan.n_matrices,), -1.0, device="cuda")
    plan.orthogonalize(p, ortho, None, res)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
    plan.compose(ortho, kf, kb)
    plan.check()
    return plan, mats, ortho, res, kf, kb


def check_construction(plan, mats, ortho, res, kf, layers):
    o_ortho, _, o_k = oracle_construct(layers, mats)
    ortho_h = ortho.cpu().numpy()
    for i, X in enumerate(o_ortho):
        if X.size == 0:
            continue
        m = plan.matrices[i]
        got = ortho_h[m["off"]: m["off"] + m["m"] * m["n"]].reshape(m["m"], m["n"])
        assert rel(got, X) < TOL16, (i, m)
    kf_h = torch.from_numpy(kf.cpu().numpy())
    for l, K in enumerate(o_k):
        assert rel(plan.kernel_f32(kf_h, l).numpy(), K) < TOL16, l
    assert float(res.max()) < 1e-3
    return o_k


def check_layer_output(plan, kb, l, d, o_kl, xin, got, H):
    """Frobenius vs the oracle conv with the ORACLE's kernel (construction + conv errors, TOL16), and
    elementwise vs the oracle conv with the GPU's own BF16 kernel (the conv alone, tight bound)."""
    assert rel(got, oracle_apply(d, o_kl, xin, H)) < TOL16, l
    kg = plan.kernel_bf16(kb, l).float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2)
    ref = oracle_apply(d, kg, xin, H)
    absref = oracle_apply(d, np.abs(kg), np.abs(xin), H)
    assert rel(got, ref) < 1e-2, l
    assert_elementwise(got, ref, absref, *BF16_ELEM, what=f"layer {l}")


def oracle_apply(d, K, x_nhwc, H):
    """Oracle forward of one layer (transposed: the adjoint onto the large grid)."""
    OL = oracle_layer(d)
    x = nchw(np.asarray(x_nhwc, np.float64))
    if d["kind"] == "convT":
        return nhwc(O.conv_transpose2d(x, K, H * d["s"], H * d["s"], s=OL.s, d=OL.d, g=OL.g, mode=OL.padding_mode))
    return nhwc(O.conv2d(x, K, s=OL.s, d=OL.d, g=OL.g, mode=OL.padding_mode))


def test_cfg3_fullsize(cuda_lib):
    """ImageNet AOC-ResNet34 shape: 33 layers, batch 256 at 224x224, chained."""
    layers = configs.cfg3()
    N = configs.BATCH[3]
    plan, mats, ortho, res, kf, kb = construct_bf16(cuda_lib, layers, 3, max_batch=N)
    o_k = check_construction(plan, mats, ortho, res, kf, layers)
    x = gen.bf16_round(gen.activations((N, 224, 224, 3), (3, 0, 0, 0, gen.ROLE_ID["x"])))
    cur, H = dev(x, torch.bfloat16), 224
    sample = [0, N - 1]
    for l, d in enumerate(layers):
        Ho, _ = plan.out_hw(l, H, H)
        y = torch.empty((N, Ho, Ho, d["c_out"]), device="cuda", dtype=torch.bfloat16)
        plan.conv_forward(l, plan.kernel_bf16(kb, l), cur, y)
        xin = cur[sample].float().cpu().numpy()
        check_layer_output(plan, kb, l, d, o_k[l], xin, y[sample].float().cpu().numpy(), H)
        cur, H = y, Ho
    plan.check()


def test_cfg4_fullsize(cuda_lib):
    """1024-channel paths at 56x56, batch 256: g32, d2, s2, transposed s2,
    transposed g32 d2 (each layer fed its own seeded input, as in bench.py)."""
    layers = configs.cfg4()
    N = configs.BATCH[4]
    plan, mats, ortho, res, kf, kb = construct_bf16(cuda_lib, layers, 4, max_batch=N)
    o_k = check_construction(plan, mats, ortho, res, kf, layers)
    sample = [0, N - 1]
    for l, d in enumerate(layers):
        H = d["H"]
        x = gen.bf16_round(gen.activations((N, H, H, d["c_in"]), (4, 0, l, 0, gen.ROLE_ID["x"])))
        xd = dev(x, torch.bfloat16)
        if d["kind"] == "convT":
            y = torch.empty((N, H * d["s"], H * d["s"], d["c_out"]), device="cuda", dtype=torch.bfloat16)
            plan.conv_transpose(l, plan.kernel_bf16(kb, l), xd, y)
        else:
            Ho, _ = plan.out_hw(l, H, H)
            y = torch.empty((N, Ho, Ho, d["c_out"]), device="cuda", dtype=torch.bfloat16)
            plan.conv_forward(l, plan.kernel_bf16(kb, l), xd, y)
        check_layer_output(plan, kb, l, d, o_k[l], x[sample], y[sample].float().cpu().numpy(), H)
        del xd, y
        torch.cuda.empty_cache()
    plan.check()


@pytest.mark.parametrize("n", [2048, 4096, 8192])
def test_cfg5_sweep(cuda_lib, n):
    """64 dense n x n matrices (OrthoLinear weights) in one batched NS: every
    residual |I - X^T X|_F <= 1e-3 on the GPU; at n = 2048 one matrix is also
    compared with the float64 oracle (the oracle cannot afford all 64)."""
    layers = configs.cfg5(n)
    plan = cuda_lib.Plan(layers, 0, compute="bf16")
    params = torch.zeros(plan.params_numel, device="cuda")
    for i, m in enumerate(plan.matrices):
        key = (5, m["layer"], m["group"], i, gen.ROLE_ID[m["role"]])
        params[m["off"]: m["off"] + m["m"] * m["n"]] = gen.param_matrix_torch(m["m"], m["n"], key, torch,
                                                                                torch.device("cuda")).ravel()
    ortho = torch.zeros_like(params)
    res = torch.full((plan.n_matrices,), -1.0, device="cuda")
    plan.orthogonalize(params, ortho, None, res)
    plan.check()
    assert float(res.min()) >= 0.0 and float(res.max()) < 1e-3
    if n == 2048:
        m = plan.matrices[0]
        W = params[m["off"]: m["off"] + n * n].reshape(n, n).cpu().numpy()
        (X,), _ = O.orthogonalize([W], T=12, beta=0.5, prescale="power", P=3)   # v0 = ones / sqrt(n), as the GPU
        got = ortho[m["off"]: m["off"] + n * n].reshape(n, n).cpu().numpy()
        assert rel(got, X) < TOL16
    del params, ortho
    torch.cuda.empty_cache()
