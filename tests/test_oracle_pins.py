"""Pins of the float64 oracle against what the paper and mathematics fix
(closed forms, library routines, brute force on tiny inputs, invariants,
SPEC worked examples).  CPU only.  Each test names the oracle step it pins.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
from synth import configs, gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
rs = np.random.default_rng(1234)


def t64(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64))


# --------------------------------------------------------------------- O2
def test_prescale_special_cases():
    W0, sig, _ = O.prescale_power(np.array(GOLD["power_identity"]["W"], float), 3, np.ones(3) / math.sqrt(3))
    assert abs(sig - 1.0) < 1e-15 and np.allclose(W0, np.eye(3), atol=1e-15)
    g = GOLD["power_diag21"]
    W0, sig, _ = O.prescale_power(np.array(g["W"], float), 60, np.ones(2) / math.sqrt(2))
    assert abs(sig - g["sigma"]) < 1e-12
    assert np.allclose(W0, np.array(g["W0"]), atol=1e-12)


def test_prescale_matches_lapack_sigma_max():
    # 50 iterations -> sigma_max of the SVD (LAPACK) to 1e-6
    for shape in [(8, 8), (12, 5), (5, 12)]:
        W = rs.standard_normal(shape)
        v = rs.standard_normal(shape[1]); v /= np.linalg.norm(v)
        _, sig, vn = O.prescale_power(W, 50, v)
        smax = np.linalg.svd(W, compute_uv=False)[0]
        assert abs(sig - smax) / smax < 1e-6
        assert abs(np.linalg.norm(vn) - 1) < 1e-12


def test_prescale_zero_and_frobenius():
    with pytest.raises(ZeroDivisionError):
        O.prescale_power(np.zeros((3, 3)), 3, np.ones(3))
    W = rs.standard_normal((7, 4))
    W0, f = O.prescale_frobenius(W)
    sv = np.linalg.svd(W, compute_uv=False)
    # |W|_F is the 2-norm of the singular values (LAPACK, independent of the oracle's sum of squares)
    assert abs(f - np.sqrt((sv ** 2).sum())) < 1e-12
    assert np.linalg.svd(W0, compute_uv=False)[0] <= 1.0
    # W0 itself: unit Frobenius norm and W0 * f reproduces W -- W / f^2 fails both
    assert abs(np.linalg.norm(W0, "fro") - 1.0) < 1e-14
    assert np.allclose(W0 * f, W, rtol=0, atol=1e-14)
    # by hand: [[3, 4], [0, 0]] -> f = 5, W0 = [[0.6, 0.8], [0, 0]]
    W0h, fh = O.prescale_frobenius(np.array([[3.0, 4.0], [0.0, 0.0]]))
    assert fh == 5.0 and np.allclose(W0h, [[0.6, 0.8], [0.0, 0.0]], rtol=0, atol=1e-16)


def test_power_iteration_one_step_by_hand():
    # one step from v = e1 on W = [[3, 4], [0, 0]]: Wv = (3, 0) -> u = e1; w = W^T u = (3, 4); sig = 5
    _, sig, v = O.prescale_power(np.array([[3.0, 4.0], [0.0, 0.0]]), 1, np.array([1.0, 0.0]))
    assert abs(sig - 5.0) < 1e-15 and np.allclose(v, [0.6, 0.8])


# --------------------------------------------------------------------- O3
def _closed_form(W0, T, beta):
    U, S, Vt = np.linalg.svd(W0, full_matrices=False)
    for _ in range(T):
        S = (1 + beta) * S - beta * S ** 3
    return (U * S) @ Vt


@pytest.mark.parametrize("shape", [(16, 16), (24, 9), (9, 24), (40, 40)])
@pytest.mark.parametrize("beta", [0.5, 0.3])
def test_bjorck_closed_form(shape, beta):
    # NS_T(W0) = U f^T(Sigma) V^T with f(s) = (1+beta)s - beta s^3 (SURVEY §8(c) O3 pin)
    W = rs.standard_normal(shape)
    W0 = W / np.linalg.svd(W, compute_uv=False)[0] * 0.97
    for T in (1, 2, 5, 12):
        X = O.bjorck(W0, T, beta)
        Y = _closed_form(W0, T, beta)
        assert np.abs(X - Y).max() < 1e-12, (T, np.abs(X - Y).max())


def test_bjorck_converges_to_polar_and_fixed_points():
    W = rs.standard_normal((20, 12))
    W0 = W / np.linalg.svd(W, compute_uv=False)[0]
    U, _, Vt = np.linalg.svd(W0, full_matrices=False)
    X = O.bjorck(W0, 60, 0.5)
    assert np.abs(X - U @ Vt).max() < 1e-10              # S:129 polar factor
    assert np.abs(O.bjorck(np.eye(6), 12) - np.eye(6)).max() == 0.0
    Q, _ = np.linalg.qr(rs.standard_normal((9, 9)))
    assert np.abs(O.bjorck(Q, 12) - Q).max() < 1e-14


def test_bjorck_residual_monotone():
    # |W_t^T W_t - I| non-increasing when |W0|_2 <= 1
    W = rs.standard_normal((30, 30))
    X = W / np.linalg.svd(W, compute_uv=False)[0]
    prev = O.ns_residual(X)
    for _ in range(25):
        X = O.bjorck(X, 1)
        r = O.ns_residual(X)
        assert r <= prev + 1e-14
        prev = r


def test_orthogonalize_near_orthogonal_T12():
    # R21: near-orthogonal parameters converge in 12 iterations ("12-25")
    for (m, n) in [(64, 64), (128, 64), (64, 256)]:
        W = gen.param_matrix(m, n, (9, m, n, 0, 1)).astype(np.float64)
        (X,), _ = O.orthogonalize([W], T=12)
        assert O.ns_residual(X) < 1e-10


# --------------------------------------------------------------------- O4
def test_block_conv_identity_and_matmul():
    g = GOLD["blockconv_1x1"]
    A = np.array(g["A"], float)[:, :, None, None]
    B = np.array(g["B"], float)[:, :, None, None]
    assert np.array_equal(O.block_conv(A, B)[:, :, 0, 0], np.array(g["AB"], float))
    K = rs.standard_normal((3, 4, 3, 2))
    delta_r = np.eye(4)[:, :, None, None]
    delta_l = np.eye(3)[:, :, None, None]
    assert np.array_equal(O.block_conv(K, delta_r), K)
    assert np.array_equal(O.block_conv(delta_l, K), K)


@pytest.mark.parametrize("k1,k2", [((2, 2), (2, 2)), ((3, 1), (2, 3)), ((1, 1), (3, 3))])
def test_block_conv_is_composition_torch(k1, k2):
    # conv_{K1}(conv_{K2}(x)) = conv_{K1 (*) K2}(x) (zero padding, summed pads);
    # checked with torch-CPU f64 conv2d, an independent library routine
    K1 = rs.standard_normal((3, 4, *k1))
    K2 = rs.standard_normal((4, 2, *k2))
    x = rs.standard_normal((2, 2, 9, 8))
    seq = F.conv2d(F.conv2d(t64(x), t64(K2), padding=(k2[0] - 1, k2[1] - 1)), t64(K1),
                   padding=(k1[0] - 1, k1[1] - 1))
    K = O.block_conv(K1, K2)
    fused = F.conv2d(t64(x), t64(K), padding=(k1[0] + k2[0] - 2, k1[1] + k2[1] - 2))
    assert torch.allclose(seq, fused, atol=1e-10)


def test_block_conv_circular_composition_and_stride():
    # composition under circular padding with a strided outer conv (the AOC use)
    K1 = rs.standard_normal((5, 3, 2, 2))   # outer, stride 2
    K2 = rs.standard_normal((3, 3, 2, 2))   # inner, stride 1
    x = rs.standard_normal((1, 3, 8, 8))
    xt = t64(x)
    inner = F.conv2d(F.pad(xt, (0, 1, 0, 1), mode="circular"), t64(K2))
    outer = F.conv2d(F.pad(inner, (0, 1, 0, 1), mode="circular"), t64(K1), stride=2)
    K = O.block_conv(K1, K2)
    fused = F.conv2d(F.pad(xt, (0, 2, 0, 2), mode="circular"), t64(K), stride=2)
    assert torch.allclose(outer, fused, atol=1e-10)


def test_block_conv_associative():
    A = rs.standard_normal((2, 3, 2, 1)); B = rs.standard_normal((3, 4, 1, 2)); C = rs.standard_normal((4, 2, 2, 2))
    assert np.abs(O.block_conv(O.block_conv(A, B), C) - O.block_conv(A, O.block_conv(B, C))).max() < 1e-12


# --------------------------------------------------------------------- O5
def _proj(c, r):
    U, _ = np.linalg.qr(rs.standard_normal((c, r)))
    return U @ U.T, U


def test_block_orth_unitary_symbol_and_factorisation():
    Pa, _ = _proj(6, 3); Pb, _ = _proj(6, 3)
    K = O.block_orth(Pa, Pb)
    I = np.eye(6)
    H = np.stack([Pa, I - Pa], -1)[:, :, :, None]      # 2x1 vertical [Pa; I-Pa]
    W = np.stack([Pb, I - Pb], -1)[:, :, None, :]      # 1x2 horizontal [Pb | I-Pb]
    assert np.abs(O.block_conv(H, W) - K).max() < 1e-14
    for _ in range(5):
        z1, z2 = np.exp(2j * np.pi * rs.random(2))
        M = K[:, :, 0, 0] + K[:, :, 0, 1] * z2 + K[:, :, 1, 0] * z1 + K[:, :, 1, 1] * z1 * z2
        assert np.abs(M.conj().T @ M - I).max() < 1e-13


def test_bcop_degenerate_and_orthogonal():
    Q, _ = np.linalg.qr(rs.standard_normal((4, 4)))
    assert np.array_equal(O.bcop(Q, [], 4, 4)[:, :, 0, 0], Q)        # S:235 k'=1 -> Q
    Us = [_proj(4, 2)[1] for _ in range(4)]
    K = O.bcop(Q, Us, 4, 4)
    assert K.shape == (4, 4, 3, 3)
    T = O.toeplitz(lambda x: O.conv2d(x, K), (4, 8, 8))
    sv = np.linalg.svd(T, compute_uv=False)
    assert np.abs(sv - 1).max() < 1e-12


# --------------------------------------------------------------------- O6
def test_rko_equals_pixel_unshuffle_matmul():
    # stride-s RKO conv == pixel_unshuffle + 1x1 conv with R (torch library)
    co, cm, s = 6, 3, 2
    R = rs.standard_normal((co, cm * s * s))
    K = O.rko(R, co, cm, s)
    x = rs.standard_normal((2, cm, 8, 8))
    y = O.conv2d(x, K, s=s, mode="circular")
    ref = F.conv2d(F.pixel_unshuffle(t64(x), s), t64(R)[:, :, None, None])
    assert np.abs(y - ref.numpy()).max() < 1e-12


# --------------------------------------------------------------------- O8/O9
@pytest.mark.parametrize("s,d,g,k,mode", [(1, 1, 1, 3, "zeros"), (2, 1, 1, 3, "zeros"), (1, 2, 2, 3, "zeros"),
                                          (2, 3, 1, 3, "circular"), (1, 1, 2, 2, "circular"),
                                          (3, 1, 1, 4, "circular"), (2, 1, 1, 5, "circular")])
def test_conv2d_matches_torch(s, d, g, k, mode):
    x = rs.standard_normal((2, 4, 12, 11))
    K = rs.standard_normal((6, 4 // g, k, k))
    e = d * (k - 1); pads = (e // 2, e - e // 2, e // 2, e - e // 2)
    y = O.conv2d(x, K, s=s, d=d, g=g, pads=pads, mode=mode)
    xp = F.pad(t64(x), (pads[2], pads[3], pads[0], pads[1]), mode="circular" if mode == "circular" else "constant")
    ref = F.conv2d(xp, t64(K), stride=s, dilation=d, groups=g)
    assert y.shape == tuple(ref.shape)
    assert np.abs(y - ref.numpy()).max() < 1e-12


def test_conv2d_spec_examples():
    for key in ("conv_identity_1x1", "conv_center_delta"):
        g = GOLD[key]
        x = rs.standard_normal((1, 1, g["H"], g["H"]))
        y = O.conv2d(x, np.array(g["kernel"], float), s=g["s"], pads=tuple(g["pads"]), mode="zeros")
        assert np.array_equal(y, x)
    g = GOLD["conv_ones_stride2"]
    y = O.conv2d(np.array(g["input"], float), np.array(g["kernel"], float), s=2, pads=(0, 0, 0, 0), mode="zeros")
    assert np.array_equal(y, np.array(g["expect"], float))
    g = GOLD["convT_ones_stride2"]
    x = O.conv_transpose2d(np.array(g["input"], float), np.array(g["kernel"], float), 4, 4, s=2,
                           pads=(0, 0, 0, 0), mode="zeros")
    assert np.array_equal(x, np.array(g["expect"], float))


@pytest.mark.parametrize("s,d,g,k,mode,H", [(1, 1, 1, 3, "circular", 8), (2, 1, 1, 3, "zeros", 9),
                                            (2, 3, 2, 3, "circular", 12), (2, 1, 1, 4, "zeros", 8),
                                            (1, 2, 1, 3, "zeros", 7), (3, 1, 1, 3, "circular", 9)])
def test_conv_transpose_adjoint(s, d, g, k, mode, H):
    K = rs.standard_normal((4, 6 // g, k, k))
    x = rs.standard_normal((2, 6, H, H))
    y = O.conv2d(x, K, s=s, d=d, g=g, mode=mode)
    yr = rs.standard_normal(y.shape)
    xt = O.conv_transpose2d(yr, K, H, H, s=s, d=d, g=g, mode=mode)
    lhs, rhs = float((y * yr).sum()), float((x * xt).sum())
    assert abs(lhs - rhs) < 1e-11 * max(1.0, abs(lhs))


def test_conv_transpose_matches_torch_zero_padding():
    K = rs.standard_normal((4, 3, 3, 3))
    H = 9
    y = rs.standard_normal((2, 4, 5, 5))          # conv of 9x9 with s=2 same-pad (1,1)
    x = O.conv_transpose2d(y, K, H, H, s=2, pads=(1, 1, 1, 1), mode="zeros")
    ref = F.conv_transpose2d(t64(y), t64(K), stride=2, padding=1, output_padding=0)
    assert np.abs(x - ref.numpy()).max() < 1e-12


# --------------------------------------------------------------------- O10
def test_toeplitz_reproduces_conv_and_fft():
    K = rs.standard_normal((3, 2, 3, 3))
    T = O.toeplitz(lambda x: O.conv2d(x, K, d=2), (2, 8, 8))
    x = rs.standard_normal((2, 8, 8))
    assert np.abs(T @ x.ravel() - O.conv2d(x[None], K, d=2).ravel()).max() < 1e-12
    sv_t = np.sort(np.linalg.svd(T, compute_uv=False))
    sv_f = O.fft_singular_values(K, 8, 8, d=2)
    sv_f = sv_f[-len(sv_t):]
    assert np.abs(sv_t - sv_f).max() < 1e-10


@pytest.mark.parametrize("co,ci,k,s,H", [(4, 8, 3, 2, 8), (3, 5, 4, 2, 8), (2, 6, 3, 3, 9), (4, 3, 5, 2, 10)])
def test_polyphase_equals_toeplitz(co, ci, k, s, H):
    K = rs.standard_normal((co, ci, k, k))
    T = O.toeplitz(lambda x: O.conv2d(x, K, s=s), (ci, H, H))
    sv_t = np.sort(np.linalg.svd(T, compute_uv=False))
    sv_p = O.polyphase_singular_values(K, H, H, s)
    sv_p = sv_p[-len(sv_t):]
    assert np.abs(sv_t - sv_p).max() < 1e-10


# --------------------------------------------------------------------- O7 + whole path
def _exact_ortho_mats(L):
    """Exactly (semi-)orthogonal matrices of the layer's shapes (QR), to pin the
    composition independently of Bjorck."""
    out = []
    for _ in range(L.g):
        ms = []
        for M in O.layer_matrices(L):
            if M.n == 0:
                ms.append(np.zeros((M.m, 0)))
                continue
            A = rs.standard_normal((max(M.m, M.n), min(M.m, M.n)))
            Q, _ = np.linalg.qr(A)
            ms.append(Q if M.m >= M.n else Q.T)
        out.append(ms)
    return out


AOC_GRID = [  # (c_in, c_out, k, s, d, g, kind)
    (16, 16, 3, 1, 1, 1, "conv"), (4, 4, 3, 1, 1, 1, "conv"), (4, 8, 3, 1, 1, 1, "conv"), (8, 4, 3, 1, 1, 1, "conv"),
    (4, 4, 2, 1, 1, 1, "conv"), (4, 4, 5, 1, 1, 1, "conv"), (4, 4, 4, 1, 1, 1, "conv"), (4, 8, 3, 2, 1, 1, "conv"),
    (8, 4, 3, 2, 1, 1, "conv"), (4, 4, 3, 2, 1, 1, "conv"), (1, 8, 3, 2, 1, 1, "conv"), (2, 8, 3, 2, 1, 1, "conv"),
    (4, 16, 3, 2, 1, 1, "conv"), (4, 32, 3, 2, 1, 1, "conv"), (8, 8, 4, 2, 1, 1, "conv"), (4, 4, 2, 2, 1, 1, "conv"),
    (4, 16, 2, 2, 1, 1, "conv"), (1, 4, 2, 2, 1, 1, "conv"), (4, 4, 1, 1, 1, 1, "conv"), (1, 1, 3, 1, 1, 1, "conv"),
    (8, 8, 3, 1, 1, 2, "conv"), (8, 16, 3, 2, 1, 2, "conv"), (4, 4, 3, 1, 2, 1, "conv"), (4, 8, 3, 2, 3, 1, "conv"),
    (8, 8, 3, 1, 2, 2, "convT"), (8, 4, 3, 2, 1, 1, "convT"), (4, 8, 3, 2, 1, 2, "convT"), (4, 4, 3, 1, 1, 1, "convT"),
]


@pytest.mark.parametrize("ci,co,k,s,d,g,kind", AOC_GRID)
def test_aoc_orthogonal_toeplitz(ci, co, k, s, d, g, kind):
    # P:330 "rigorously proven orthogonal for any valid configuration (k >= s)";
    # P:462 Toeplitz SVD on small images; all min(rows, cols) sigma = 1 (R9, R12)
    L = O.Layer(ci, co, k, s, d, g, kind=kind)
    K = O.layer_kernel(L, _exact_ortho_mats(L))
    ci_f, co_f = L.fwd_channels()
    assert K.shape == (co_f, ci_f // g, k, k)
    H = 12 if s == 3 or d == 3 else 8
    if kind == "conv":
        op, shape = (lambda x: O.conv2d(x, K, s=s, d=d, g=g)), (ci_f, H, H)
    else:
        Hs = H // s
        op, shape = (lambda y: O.conv_transpose2d(y, K, H, H, s=s, d=d, g=g)), (co_f, Hs, Hs)
    T = O.toeplitz(op, shape)
    sv = np.linalg.svd(T, compute_uv=False)
    r = min(T.shape)
    assert np.abs(sv[:r] - 1).max() < 1e-10, (sv.min(), sv.max())
    if kind == "conv":   # scalable estimator agrees with the exact one
        sv2 = O.conv_singular_values(K, L, H, H)
        assert np.abs(sv2[-r:] - 1).max() < 1e-10


def test_zero_padding_is_one_lipschitz_only():
    # R12: zero padding -> sigma_max <= 1 (no lower bound); P:462 tests transposed with zero padding only
    L = O.Layer(4, 4, 3, 1, padding_mode="zeros")
    K = O.layer_kernel(L, _exact_ortho_mats(L))
    T = O.toeplitz(lambda x: O.conv2d(x, K, mode="zeros"), (4, 8, 8))
    sv = np.linalg.svd(T, compute_uv=False)
    assert sv.max() <= 1 + 1e-12 and sv.min() < 0.5


def test_gcd_stride_dilation_breaks_orthogonality():
    # R10: gcd(s, d) != 1 loses orthogonality (why the boundary rejects it)
    L = O.Layer(4, 8, 3, 2, 2)
    K = O.layer_kernel(L, _exact_ortho_mats(L))
    sv = O.conv_singular_values(K, L, 8, 8)
    assert sv.max() > 1.2


def test_cfg1_whole_path_norm_preservation():
    # whole path on cfg1: params -> power/Bjorck -> BCOP -> conv; |y| = |x| per sample (isometry)
    Ld = configs.cfg1()[0]
    L = O.Layer(Ld["c_in"], Ld["c_out"], Ld["k"], Ld["s"], Ld["d"], Ld["g"])
    specs = O.layer_matrices(L)
    mats = [gen.param_matrix(M.m, M.n, (1, 0, 0, j, gen.ROLE_ID[M.role])).astype(np.float64)
            for j, M in enumerate(specs)]
    ortho, _ = O.orthogonalize(mats, T=12)
    for X in ortho:
        assert O.ns_residual(X) < 1e-12
    K = O.layer_kernel(L, [ortho])
    x = gen.activations((2, 16, 8, 8), (1, 0, 0, 0, gen.ROLE_ID["x"])).astype(np.float64)
    y = O.conv2d(x, K)
    nx = np.sqrt((x ** 2).sum(axis=(1, 2, 3)))
    ny = np.sqrt((y ** 2).sum(axis=(1, 2, 3)))
    assert np.abs(ny / nx - 1).max() < 1e-12


# --------------------------------------------------------------------- a1 derivation
def _count(cfg_layers):
    n, flops = 0, 0.0
    for Ld in cfg_layers:
        L = O.Layer(Ld["c_in"], Ld["c_out"], Ld["k"], Ld["s"], Ld["d"], Ld["g"], kind=Ld["kind"])
        for M in O.layer_matrices(L):
            n += L.g
            m_, n_ = max(M.m, M.n), min(M.m, M.n)
            flops += L.g * 4.0 * m_ * n_ * n_ * 12
    return n, flops


def test_unit_derivation_counts_match_survey():
    # SURVEY §8(d) totals: cfg2 57 matrices / 45.5 GF; cfg3 158 / 99.8 GF; cfg4 333 / 670 GF (T = 12)
    n2, f2 = _count(configs.cfg2())
    n3, f3 = _count(configs.cfg3())
    n4, f4 = _count(configs.cfg4())
    assert (n2, n3, n4) == (57, 158, 333)
    assert abs(f2 / 1e9 - 45.5) < 0.1 and abs(f3 / 1e9 - 99.8) < 0.1 and abs(f4 / 1e9 - 670) < 1.0


# ------------------------------------------------------------------ f2: spectral certificate
@pytest.mark.parametrize("ci,co,k,s,d,g,H", [(4, 4, 3, 1, 1, 1, 6), (3, 5, 3, 2, 1, 1, 8), (6, 4, 4, 2, 1, 2, 8),
                                           (4, 8, 3, 2, 1, 1, 8), (2, 3, 3, 1, 2, 1, 7)])
def test_spectral_certificate_against_toeplitz(ci, co, k, s, d, g, H):
    """Brute force on tiny inputs: the Toeplitz matrix T of the circular operator (impulse responses, no
    symbol code involved) fixes (i) max_f |E_f|_2 = max |sigma^2 - 1| over the singular values of T on the
    short side, and (ii) sum_f |E_f|_F^2 = |T^T T - I|_F^2 (input short side) or |T T^T - I|_F^2 (output
    short side): the per-frequency block diagonalisation is unitary, so Frobenius norms add up exactly."""
    L = O.Layer(ci, co, k, s, d, g)
    K = rs.standard_normal((co, ci // g, k, k)) * 0.3
    frob, spec, sig_dev = O.spectral_certificate(K, L, H, H)
    T = O.toeplitz(lambda x: O.conv2d(x, K, s=s, d=d, g=g), (ci, H, H))
    sv = np.linalg.svd(T, compute_uv=False)
    short = min(T.shape)
    dev2 = np.abs(sv[:short] ** 2 - 1)
    if T.shape[0] >= T.shape[1]:
        G = T.T @ T
    else:
        G = T @ T.T
    assert abs(spec.max() - dev2.max()) < 1e-10 * max(1.0, dev2.max())
    assert abs((frob ** 2).sum() - np.linalg.norm(G - np.eye(G.shape[0])) ** 2) < 1e-9 * max(1.0, (frob ** 2).sum())
    assert abs(sig_dev - np.abs(sv[:short] - 1).max()) < 1e-10
    assert (frob >= spec - 1e-12).all()                      # |E|_F >= |E|_2: the certificate is an upper bound


def test_spectral_certificate_orthogonal_and_dense():
    """An AOC kernel built by the oracle is orthogonal: every |E_f|_F ~ 1e-15 (P:462 tolerance 1e-4 is met by
    11 orders of magnitude); a dense orthogonal matrix has one frequency with |E|_F ~ 0, and 2 I gives
    E = 3 I, |E|_F = 3 sqrt(n)."""
    L = O.Layer(8, 16, 3, 2)
    ms = [gen.param_matrix(M.m, M.n, (99, 0, 0, i, 1)).astype(np.float64) for i, M in enumerate(O.layer_matrices(L))]
    ortho, _ = O.orthogonalize(ms, T=25)
    K = O.layer_kernel(L, [ortho])
    frob, spec, sig_dev = O.spectral_certificate(K, L, 8, 8)
    assert frob.max() < 1e-12 and sig_dev < 1e-12
    Ld = O.Layer(5, 5, 1, kind="dense")
    frob, spec, _ = O.spectral_certificate(2 * np.eye(5), Ld, 1, 1)
    assert frob.shape == (1, 1, 1) and abs(frob[0, 0, 0] - 3 * np.sqrt(5)) < 1e-12 and abs(spec[0, 0, 0] - 3) < 1e-12


# ------------------------------------------------------------------ f3: SOC explicit exponential
def _circ(K, x, d=1):
    """torch-CPU f64 circular 'same' conv (independent of the oracle's conv2d)."""
    k = K.shape[2]
    p = d * (k - 1) // 2
    xt = F.pad(t64(x), (p, p, p, p), mode="circular")
    return F.conv2d(xt, t64(K), dilation=d).numpy()


def test_soc_degenerate_cases():
    """K = 0 -> the identity kernel; a symmetric free kernel (K[a,b,i,j] = K[b,a,k-1-i,k-1-j]) has a
    zero skew part -> identity."""
    E, _ = O.soc_exp_kernel(np.zeros((3, 3, 3, 3)), 4)
    I = np.zeros((3, 3, 9, 9)); I[:, :, 4, 4] = np.eye(3)
    assert np.array_equal(E, I)
    A = rs.standard_normal((3, 3, 3, 3))
    S = A + np.transpose(A, (1, 0, 2, 3))[:, :, ::-1, ::-1]
    assert np.abs(O.soc_skew(S)).max() < 1e-15
    E, _ = O.soc_exp_kernel(S, 3)
    assert np.abs(E - I[:, :, 1:8, 1:8]).max() < 1e-15


@pytest.mark.parametrize("c,k,d", [(4, 3, 1), (3, 5, 1), (4, 3, 2)])
def test_soc_skew_adjoint_and_aol_bound(c, k, d):
    """Toeplitz brute force: T(soc_skew(K)) is skew (T^T = -T) on a circular grid, and the AOL scalar makes
    |T(alpha L)|_2 <= 1 (S:274 certified upper bound)."""
    K = rs.standard_normal((c, c, k, k))
    L = O.soc_skew(K)
    H = 2 * d * (k - 1) + 3
    T = O.toeplitz(lambda x: _circ(L, x, d), (c, H, H))
    assert np.abs(T + T.T).max() < 1e-12
    a = O.aol_scale(L)
    assert np.linalg.svd(a * T, compute_uv=False)[0] <= 1 + 1e-12
    # 1x1 kernel = 2I -> d_i = 4 -> alpha = 1/2
    assert abs(O.aol_scale(2 * np.eye(3)[:, :, None, None]) - 0.5) < 1e-15


@pytest.mark.parametrize("c,k,terms,d", [(4, 3, 6, 1), (3, 3, 8, 2), (2, 5, 4, 1)])
def test_soc_explicit_equals_implicit_and_expm(c, k, terms, d):
    """the explicit kernel applied once equals the implicit series x + L*x + L*L*x/2! + ... applied
    term by term (torch-CPU conv, S:266 example), and its circular operator equals the truncated matrix
    exponential sum_j T(L)^j / j! of the Toeplitz matrix (brute force); against scipy's expm of T(L) it is
    off only by the tail bound e |T(L)|^{n+1} / (n+1)!, so it is orthogonal to that accuracy."""
    import scipy.linalg
    K = rs.standard_normal((c, c, k, k))
    E, alpha = O.soc_exp_kernel(K, terms)
    L = alpha * O.soc_skew(K)
    Hx = max(10, d * (E.shape[2] - 1) // 2 + 2)
    for _ in range(3):
        x = rs.standard_normal((1, c, Hx, Hx))
        imp, term = x.copy(), x.copy()
        for j in range(1, terms + 1):
            term = _circ(L, term, d) / j
            imp = imp + term
        assert np.abs(_circ(E, x, d) - imp).max() < 1e-10 * max(1.0, np.abs(imp).max())
    H = max(7, d * (E.shape[2] - 1) // 2 + 2)
    TL = O.toeplitz(lambda z: _circ(L, z, d), (c, H, H))
    TE = O.toeplitz(lambda z: _circ(E, z, d), (c, H, H))
    acc, P = np.eye(TL.shape[0]), np.eye(TL.shape[0])
    for j in range(1, terms + 1):
        P = P @ TL / j
        acc = acc + P
    assert np.abs(TE - acc).max() < 1e-11
    nrm = np.linalg.svd(TL, compute_uv=False)[0]
    assert nrm <= 1 + 1e-12
    tail = math.e * nrm ** (terms + 1) / math.factorial(terms + 1)
    assert np.linalg.norm(TE - scipy.linalg.expm(TL), 2) <= tail + 1e-12
    sv = np.linalg.svd(TE, compute_uv=False)
    assert np.abs(sv - 1).max() <= tail + 1e-12


# ------------------------------------------------------------------ f4: SLL x AOC block
def test_aol_rescale_bound_and_examples():
    """the rescaled operator has Toeplitz sigma_max <= 1; 1x1 I unchanged, 2I -> I; a zero input
    channel passes unscaled."""
    for shape in [(4, 4, 3, 3), (3, 5, 2, 2), (6, 2, 3, 3)]:
        K = O.aol_rescale(rs.standard_normal(shape))
        T = O.toeplitz(lambda x: _circ_pad(K, x), (shape[1], 7, 7))
        assert np.linalg.svd(T, compute_uv=False)[0] <= 1 + 1e-12
    I = np.eye(3)[:, :, None, None]
    assert np.array_equal(O.aol_rescale(I), I) and np.allclose(O.aol_rescale(2 * I), I, rtol=0, atol=1e-15)
    Z = rs.standard_normal((3, 3, 3, 3)); Z[:, 1] = 0
    assert np.abs(O.aol_rescale(Z)[:, 1]).max() == 0


def _circ_pad(K, x):
    """torch-CPU circular conv with the R11 'same' pads (possibly asymmetric for even k)."""
    k = K.shape[2]
    pt, pb, pl, pr = O.same_pads(k)
    return F.conv2d(F.pad(t64(x), (pl, pr, pt, pb), mode="circular"), t64(K)).numpy()


def _torch_block(x, K_pre, K_post, K, b, s):
    """The unfused block in torch (independent of the oracle's conv code): circular pad + conv, and the SLL's
    K^T * as its exact adjoint -- conv_transpose2d onto the padded grid, then the circular pad folded back."""
    def pads(k):
        return O.same_pads(k)

    def conv(z, W, stride=1):
        pt, pb, pl, pr = pads(W.shape[2])
        return F.conv2d(F.pad(z, (pl, pr, pt, pb), mode="circular"), W, stride=stride)

    def conv_adj(t, W, H):
        pt, pb, pl, pr = pads(W.shape[2])
        yp = F.conv_transpose2d(t, W)                  # (N, C, H + pt + pb, W + pl + pr)
        ri = (torch.arange(yp.shape[2]) - pt) % H
        ci = (torch.arange(yp.shape[3]) - pl) % H
        out = torch.zeros(yp.shape[0], yp.shape[1], H, yp.shape[3], dtype=yp.dtype).index_add(2, ri, yp)
        return torch.zeros(yp.shape[0], yp.shape[1], H, H, dtype=yp.dtype).index_add(3, ci, out)
    z = conv(x, t64(K_pre))
    Kt = t64(K)
    t = torch.relu(conv(z, Kt) + t64(b)[None, :, None, None])
    u = z - 2 * conv_adj(t, Kt, z.shape[2])
    return conv(u, t64(K_post), s)


@pytest.mark.parametrize("c,cs,co,kpre,ks,kpost,s,H", [(4, 6, 8, 2, 2, 3, 2, 8), (3, 3, 3, 3, 3, 3, 1, 6),
                                                       (4, 5, 6, 3, 2, 4, 2, 8), (2, 4, 8, 2, 3, 2, 2, 6)])
def test_sll_block_fused_equals_unfused(c, cs, co, kpre, ks, kpost, s, H):
    """P:392-396 / S:294-296: the fused block (merged kernels C and M = [A | -2 B]) equals the three
    sequential layers conv_{K_post, s} o SLL o conv_{K_pre} -- against the oracle's own unfused composition
    and against a torch-CPU implementation (circular pads, autograd adjoint) -- to 1e-10."""
    K_pre, K_post = rs.standard_normal((c, c, kpre, kpre)), rs.standard_normal((co, c, kpost, kpost))
    W = rs.standard_normal((cs, c, ks, ks))
    b = 0.3 * rs.standard_normal(cs)
    kern = O.sll_block_kernels(K_pre, K_post, W)
    x = rs.standard_normal((2, c, H, H))
    fused = O.sll_block_forward(x, kern, b, s)
    unf = O.sll_block_unfused(x, K_pre, K_post, kern["K"], b, s)
    ref = _torch_block(t64(x), K_pre, K_post, kern["K"], b, s).numpy()
    assert fused.shape == ref.shape
    assert np.abs(fused - unf).max() < 1e-10 * max(1.0, np.abs(unf).max())
    assert np.abs(fused - ref).max() < 1e-10 * max(1.0, np.abs(ref).max())


def test_sll_block_special_cases_and_lipschitz():
    """K = 0 -> y = (K_post (*) K_pre) *_s x; identity 1x1 K_pre / K_post at s = 1 -> the bare SLL
    layer x - 2 K^T relu(K x + b); with orthogonal K_pre / K_post the block is 1-Lipschitz: the spectral norm
    of its Jacobian (torch autograd of the torch implementation, at random points) is <= 1 + 1e-9."""
    c, cs, co = 3, 4, 6
    L = O.Layer(c, co, 3, 2)
    ms = [gen.param_matrix(M.m, M.n, (77, 0, 0, i, 1)).astype(np.float64) for i, M in enumerate(O.layer_matrices(L))]
    K_post = O.layer_kernel(L, [O.orthogonalize(ms, T=25)[0]])
    Lp = O.Layer(c, c, 2, 1)
    ms = [gen.param_matrix(M.m, M.n, (78, 0, 0, i, 1)).astype(np.float64) for i, M in enumerate(O.layer_matrices(Lp))]
    K_pre = O.layer_kernel(Lp, [O.orthogonalize(ms, T=25)[0]])
    x = rs.standard_normal((1, c, 6, 6))
    kz = O.sll_block_kernels(K_pre, K_post, np.zeros((cs, c, 2, 2)))
    y0 = O.sll_block_forward(x, kz, np.zeros(cs), 2)
    assert np.abs(y0 - O.conv2d(x, kz["A"], s=2, pads=(1, 2, 1, 2))).max() < 1e-12
    I = np.eye(c)[:, :, None, None]
    W = rs.standard_normal((cs, c, 3, 3))
    ki = O.sll_block_kernels(I, I, W)
    b = 0.1 * rs.standard_normal(cs)
    K = ki["K"]
    sll = x - 2 * O.conv_transpose2d(np.maximum(O.conv2d(x, K) + b[None, :, None, None], 0), K, 6, 6)
    assert np.abs(O.sll_block_forward(x, ki, b, 1) - sll).max() < 1e-12
    W = rs.standard_normal((cs, c, 2, 2))
    kern = O.sll_block_kernels(K_pre, K_post, W)
    b = 0.1 * rs.standard_normal(cs)
    for _ in range(3):
        x0 = t64(rs.standard_normal((1, c, 6, 6)))
        J = torch.autograd.functional.jacobian(lambda z: _torch_block(z, K_pre, K_post, kern["K"], b, 2), x0)
        J = J.reshape(-1, x0.numel()).numpy()
        assert np.linalg.svd(J, compute_uv=False)[0] <= 1 + 1e-9


# ------------------------------------------------------------------ f1: backward (VJPs) of the path
def test_conv2d_wgrad_matches_torch_and_bilinear():
    """The weight gradient against torch.nn.grad.conv2d_weight (zero padding; library routine) and the exact
    bilinear identity <dy, conv2d(x, dK)> = <wgrad(x, dy), dK> (circular, strided, dilated, grouped)."""
    for (ci, co, k, s, d, g, mode) in [(4, 6, 3, 1, 1, 1, "zeros"), (4, 6, 3, 2, 1, 2, "zeros"),
                                       (6, 4, 3, 2, 1, 1, "circular"), (4, 8, 3, 1, 2, 2, "circular")]:
        x = rs.standard_normal((2, ci, 8, 8))
        K = rs.standard_normal((co, ci // g, k, k))
        y = O.conv2d(x, K, s=s, d=d, g=g, mode=mode)
        dy = rs.standard_normal(y.shape)
        dK = O.conv2d_wgrad(x, dy, K.shape, s=s, d=d, g=g, mode=mode)
        dK2 = rs.standard_normal(K.shape)
        lhs = float((dy * O.conv2d(x, dK2, s=s, d=d, g=g, mode=mode)).sum())
        assert abs(lhs - float((dK * dK2).sum())) < 1e-10 * max(1.0, abs(lhs))
        if mode == "zeros":
            p = d * (k - 1) // 2
            ref = torch.nn.grad.conv2d_weight(t64(x), K.shape, t64(dy), stride=s, padding=p, dilation=d, groups=g)
            assert np.abs(ref.numpy() - dK).max() < 1e-10


@pytest.mark.parametrize("shape,T", [((12, 7), 5), ((7, 12), 5), ((10, 10), 12)])
def test_bjorck_vjp_finite_differences(shape, T):
    """Central finite differences of f(W0) = <G, bjorck(W0)> along random directions (float64, eps 1e-6)."""
    W = rs.standard_normal(shape)
    W0 = W / np.linalg.svd(W, compute_uv=False)[0] * 0.9
    G = rs.standard_normal(shape)
    dW = O.bjorck_vjp(W0, T, 0.5, G)
    for _ in range(3):
        D = rs.standard_normal(shape)
        eps = 1e-6
        fd = ((G * O.bjorck(W0 + eps * D, T)).sum() - (G * O.bjorck(W0 - eps * D, T)).sum()) / (2 * eps)
        assert abs(fd - (dW * D).sum()) < 1e-6 * max(1.0, abs(fd))


def test_orthogonalize_vjp_sigma_constant():
    """R31: with the pre-scale held constant the VJP is bjorck_vjp / sigma; checked by finite differences of
    W -> <G, bjorck(W / sigma_fixed)>."""
    W = gen.param_matrix(9, 6, (5, 5, 5, 0, 1)).astype(np.float64)
    G = rs.standard_normal(W.shape)
    (dW,) = O.orthogonalize_vjp([W], [G], T=8)
    W0, sig, _ = O.prescale_power(W, 3, np.ones(6) / math.sqrt(6))
    D = rs.standard_normal(W.shape)
    eps = 1e-6
    f = lambda A: (G * O.bjorck(A / sig, 8)).sum()
    assert abs((f(W + eps * D) - f(W - eps * D)) / (2 * eps) - (dW * D).sum()) < 1e-6


@pytest.mark.parametrize("ci,co,k,s,g", [(4, 4, 3, 1, 1), (4, 8, 3, 2, 1), (6, 3, 2, 1, 1), (4, 6, 4, 2, 2),
                                         (3, 8, 2, 2, 1)])
def test_layer_kernel_vjp_finite_differences(ci, co, k, s, g):
    """d<dK, layer_kernel(mats)>/d(mats) by central finite differences (BCOP chain with its projectors
    P = U U^T, RKO reshape, AOC block convolution, slicing, groups), and the block-conv adjoint identity."""
    L = O.Layer(ci, co, k, s, 1, g)
    specs = O.layer_matrices(L)
    mats = [[rs.standard_normal((M.m, M.n)) for M in specs] for _ in range(g)]
    K = O.layer_kernel(L, mats)
    dK = rs.standard_normal(K.shape)
    grads = O.layer_kernel_vjp(L, mats, dK)
    eps = 1e-6
    for gi in range(g):
        for j in range(len(specs)):
            D = rs.standard_normal(mats[gi][j].shape)
            plus = [list(m) for m in mats]; minus = [list(m) for m in mats]
            plus[gi][j] = mats[gi][j] + eps * D
            minus[gi][j] = mats[gi][j] - eps * D
            fd = ((dK * O.layer_kernel(L, plus)).sum() - (dK * O.layer_kernel(L, minus)).sum()) / (2 * eps)
            assert abs(fd - (grads[gi][j] * D).sum()) < 1e-6 * max(1.0, abs(fd)), (gi, j)
    K1, K2 = rs.standard_normal((3, 4, 2, 3)), rs.standard_normal((4, 5, 3, 2))
    dKk = rs.standard_normal((3, 5, 4, 4))
    d1, d2 = O.block_conv_vjp(K1, K2, dKk)
    E1, E2 = rs.standard_normal(K1.shape), rs.standard_normal(K2.shape)
    lin = (dKk * (O.block_conv(E1, K2) + O.block_conv(K1, E2))).sum()
    assert abs(lin - (d1 * E1).sum() - (d2 * E2).sum()) < 1e-10 * max(1.0, abs(lin))
