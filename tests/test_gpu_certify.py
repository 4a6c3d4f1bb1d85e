"""f2: GPU spectral certification against the oracle, and
the full-size orthogonality check of the BF16 hot path's kernels (north star:
max|sigma - 1| <= 1e-3; PAPER.md:208 / :462).

* parity: per (group, frequency) |E|_F of the GPU (FP64 from the FP32 kernel)
  against oracle.spectral_certificate (float64 NumPy, pinned against Toeplitz
  SVD in test_oracle_pins.py) on non-orthogonal random kernels of every layer
  shape class; the power estimate is a valid lower bound of the oracle's
  exact |E|_2 and close to it;
* full size: the FP32 kernels that orth_compose_kernel produces in BF16 mode
  (the bench's construction) for all 12 cfg2 layers and one layer per cfg3
  stage (+ the RKO stem), certified on an 8 x 8 circular grid both by the
  oracle's per-frequency SVD (max|sigma - 1| <= 1e-3) and by the GPU
  certificate (|E|_F <= 1e-3, agreeing with the oracle's |E|_F)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import configs, gen
from tests.helpers import oracle_layer, pack_params

pytestmark = pytest.mark.gpu

CASES = [  # (ci, co, k, s, d, g, kind, H)
    (8, 8, 3, 1, 1, 1, "conv", 6), (6, 12, 3, 2, 1, 1, "conv", 8), (12, 6, 3, 2, 1, 1, "conv", 8),
    (8, 8, 3, 1, 2, 2, "conv", 7), (4, 10, 5, 3, 2, 1, "conv", 9), (16, 8, 3, 2, 1, 2, "convT", 8),
    (64, 64, 3, 1, 1, 1, "conv", 8), (3, 64, 4, 4, 1, 1, "conv", 8), (40, 24, 1, 1, 1, 1, "dense", 1),
]


@pytest.mark.parametrize("case", CASES)
def test_certificate_parity(cuda_lib, case):
    ci, co, k, s, d, g, kind, H = case
    layer = dict(kind=kind, c_in=ci, c_out=co, k=k, s=s, d=d, g=g, padding_mode="circular")
    plan = cuda_lib.Plan([layer], 0)
    shape = plan.kernel_shape(0)
    K = (gen.rng(31, ci, co, k, s).standard_normal(shape) / np.sqrt(np.prod(shape[1:]))).astype(np.float32)
    out = plan.certify(0, torch.from_numpy(K).cuda().reshape(-1), H, H, power_iters=300)
    plan.check()
    got = out.cpu().numpy()
    frob, spec, _ = O.spectral_certificate(K.astype(np.float64), oracle_layer(layer), H, H)
    assert got.shape[:3] == frob.shape
    assert np.abs(got[..., 0] - frob).max() <= 1e-10 * max(1.0, frob.max())
    est = got[..., 1]
    assert (est <= spec * (1 + 1e-9) + 1e-12).all()           # a power estimate never exceeds |E|_2
    assert (est >= 0.5 * spec).all()                          # and has converged near it
    assert abs(est.max() - spec.max()) <= 1e-2 * spec.max()


def test_certificate_closed_forms(cuda_lib):
    """2 I (dense) -> E = 3 I: |E|_F = 3 sqrt(n), |E|_2 = 3 exactly; the identity kernel -> 0."""
    plan = cuda_lib.Plan([dict(kind="dense", c_in=5, c_out=5, k=1, s=1, d=1, g=1, padding_mode="circular")], 0)
    out = plan.certify(0, (2 * torch.eye(5)).cuda().reshape(-1), 1, 1, power_iters=5).cpu().numpy()
    assert abs(out[0, 0, 0, 0] - 3 * np.sqrt(5)) < 1e-12 and abs(out[0, 0, 0, 1] - 3) < 1e-12
    plan = cuda_lib.Plan([dict(kind="conv", c_in=4, c_out=4, k=3, s=1, d=1, g=1, padding_mode="circular")], 0)
    K = torch.zeros(4, 4, 3, 3)
    K[:, :, 1, 1] = torch.eye(4)
    out = plan.certify(0, K.cuda().reshape(-1), 6, 6, power_iters=5).cpu().numpy()
    assert np.abs(out).max() == 0.0


def _construct_bf16(orth, layers, cfg_id):
    plan = orth.Plan(layers, 0, compute="bf16")
    params, _ = pack_params(plan, cfg_id)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    plan.orthogonalize(p, ortho)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    plan.compose(ortho, kf)
    plan.check()
    return plan, kf


@pytest.mark.parametrize("cfg_id,which", [(2, list(range(12))), (3, [0, 1, 7, 8, 15, 16, 27, 28])])
def test_fullsize_kernels_orthogonal(cuda_lib, cfg_id, which):
    layers = configs.CONFIGS[cfg_id]()
    plan, kf = _construct_bf16(cuda_lib, layers, cfg_id)
    worst_sv, worst_cert = 0.0, 0.0
    for l in which:
        d = layers[l]
        Kdev = plan.kernel_f32(kf, l)
        K = Kdev.cpu().numpy().astype(np.float64)
        OL = oracle_layer(d)
        Hc = 8 if 8 % d["s"] == 0 else 2 * d["s"] * 2
        sv = O.conv_singular_values(K, OL, Hc, Hc)
        dev_sv = float(np.abs(sv - 1).max())
        assert dev_sv <= 1e-3, (l, dev_sv)                         # north star, oracle SVD
        out = plan.certify(l, Kdev.reshape(-1).contiguous(), Hc, Hc, power_iters=50).cpu().numpy()
        frob, spec, _ = O.spectral_certificate(K, OL, Hc, Hc)
        assert np.abs(out[..., 0] - frob).max() <= 1e-9 + 1e-9 * frob.max()
        assert out[..., 0].max() <= 1e-3, (l, out[..., 0].max())    # GPU certificate: |E|_F bounds max|s^2-1|
        assert dev_sv <= out[..., 0].max() * (1 + 1e-6) + 1e-12     # the certificate bounds the SVD's deviation
        worst_sv, worst_cert = max(worst_sv, dev_sv), max(worst_cert, float(out[..., 0].max()))
    print(f"cfg{cfg_id}: max|sigma-1| (oracle SVD) {worst_sv:.2e}, GPU certificate max|E|_F {worst_cert:.2e}")
