"""Float64 CPU oracle for the orthogonal-convolution hot path.

TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct NumPy float64.  It is
imported by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline leg, never by the product package ``paper_2601_13776_b200``, and it
imports nothing from that package (no shared kernels, headers, helpers,
constants or layouts).

Citation convention: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` =
SPEC.md line n (the SPEC binds a CPU program, we use it only for interfaces and
examples).  Where the paper is silent we follow the readings numbered R1..R21 in
DESIGN.md ("Readings of the paper"), which restate SURVEY.md §8(c).

Every function below says what it computes and the passage it follows.  Pins
that fix each function independently of itself live in ``tests/test_oracle_*.py``.
Nothing here is "parity unpinned".

Conventions (R11, R15):
  * convolution = cross-correlation, NCHW arrays, kernels (c_out, c_in/g, k, k);
  * default padding p_t = floor(d(k-1)/2), p_b = d(k-1) - p_t ("same");
  * groups are group-major along the output-channel axis (PyTorch convention);
  * parameters are ordered layer -> group -> [Q, U_1 .. U_2(k'-1), R].
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Layer", "MatrixSpec", "layer_matrices", "layer_geometry",
    "prescale_power", "prescale_frobenius", "bjorck", "ns_residual",
    "orthogonalize",
    "block_conv", "block_orth", "bcop", "rko", "layer_kernel",
    "out_size", "conv2d", "conv_transpose2d",
    "toeplitz", "fft_singular_values", "polyphase_singular_values",
    "conv_singular_values", "spectral_certificate",
    "soc_skew", "aol_scale", "soc_exp_kernel",
    "aol_rescale", "adjoint_kernel", "same_pads", "sll_block_kernels", "sll_block_forward", "sll_block_unfused",
    "conv2d_wgrad", "bjorck_vjp", "orthogonalize_vjp", "block_conv_vjp", "layer_kernel_vjp",
]


# ---------------------------------------------------------------------------
# O1/a1: layer description and unit derivation (R5-R8)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Layer:
    """One orthogonal layer.  kind: 'conv' (AdaptiveOrthoConv2d),
    'convT' (AdaptiveOrthoConvTranspose2d) or 'dense'
    (OrthoLinear weight).  padding_mode: 'circular' | 'zeros'.
    pad = (p_t, p_b, p_l, p_r) or None for the "same" rule (R11)."""
    c_in: int
    c_out: int
    k: int = 3
    s: int = 1
    d: int = 1
    g: int = 1
    kind: str = "conv"
    padding_mode: str = "circular"
    pad: Optional[Tuple[int, int, int, int]] = None
    terms: int = 6          # 'soc' (f3): highest power of the explicit exponential series

    def fwd_channels(self) -> Tuple[int, int]:
        """(c_in, c_out) of the forward conv whose kernel is built.  A
        transposed layer builds the kernel of its forward adjoint, with the
        channel counts swapped (R13)."""
        if self.kind == "convT":
            return self.c_out, self.c_in
        return self.c_in, self.c_out

    def pads(self) -> Tuple[int, int, int, int]:
        if self.pad is not None:
            return tuple(self.pad)
        ext = self.d * (self.k - 1)
        pt = ext // 2
        return (pt, ext - pt, pt, ext - pt)


@dataclass(frozen=True)
class MatrixSpec:
    """One parameter matrix: role in {'Q','U','R','W'}; shape m x n."""
    role: str
    m: int
    n: int


def layer_geometry(L: Layer) -> dict:
    """Per-group channel widths of the AOC construction.

    P:323-330 define AOC = RKO (*) K_BCOP for k >= s; the internal widths are
    not printed ("careful choice of internal channel dimensions").
    Reading R7/R8: BCOP size k' = k - s + 1; c_mid = max(ci, floor(co/s^2)).
    s == 1 -> BCOP only at width max(ci, co) (R5); k == s > 1 -> RKO only.
    """
    ci_f, co_f = L.fwd_channels()
    ci, co = ci_f // L.g, co_f // L.g
    if L.kind == "dense":
        return dict(ci=ci, co=co, kind="dense", kp=0, c_b=0, c_mid=0)
    if L.kind in ("soc", "sll", "sll_block"):
        return dict(ci=ci, co=co, kind=L.kind, kp=0, c_b=0, c_mid=0)
    if L.s == 1:
        return dict(ci=ci, co=co, kind="bcop", kp=L.k, c_b=max(ci, co), c_mid=0)
    if L.k == L.s:
        return dict(ci=ci, co=co, kind="rko", kp=0, c_b=0, c_mid=ci)
    c_mid = max(ci, co // (L.s * L.s))
    return dict(ci=ci, co=co, kind="aoc", kp=L.k - L.s + 1, c_b=c_mid, c_mid=c_mid)


def layer_matrices(L: Layer) -> List[MatrixSpec]:
    """Matrices of ONE group, in packing order [Q, U_1..U_2(k'-1), R] (R15;
    S:212-216: "BCOP: one square matrix plus 2(k-1) matrices; RKO: one matrix
    of shape c_out x (c_in s^2 / g) per group")."""
    geo = layer_geometry(L)
    if geo["kind"] == "dense":
        return [MatrixSpec("W", geo["co"], geo["ci"])]
    if geo["kind"] in ("soc", "sll"):   # f3 / f4: the free kernel (co, ci, k, k) as a co x ci k^2 matrix
        return [MatrixSpec("K", geo["co"], geo["ci"] * L.k * L.k)]
    if geo["kind"] == "sll_block":       # f4: no parameters of its own (merges three other layers)
        return []
    out: List[MatrixSpec] = []
    if geo["kind"] in ("bcop", "aoc"):
        c = geo["c_b"]
        out.append(MatrixSpec("Q", c, c))
        for _ in range(2 * (geo["kp"] - 1)):
            out.append(MatrixSpec("U", c, c // 2))          # rank floor(c/2), R5
    if geo["kind"] in ("rko", "aoc"):
        out.append(MatrixSpec("R", geo["co"], geo["c_mid"] * L.s * L.s))
    return out


# ---------------------------------------------------------------------------
# O2: pre-scaling ("spectral normalization via batched power
# iteration"; P:313 cached vector; R2/R3)
# ---------------------------------------------------------------------------
def prescale_power(W: np.ndarray, P: int, v: np.ndarray):
    """P power iterations from v: u = Wv/|Wv|; w = W^T u; sig = |w|; v = w/sig.
    Returns (W/sig, sig, v_new).  Zero W is an error."""
    W = np.asarray(W, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64).copy()
    if W.size == 0:
        return W.copy(), 0.0, v
    if not np.any(W):
        raise ZeroDivisionError("zero matrix (S:115)")
    sig = 0.0
    for _ in range(P):
        wv = W @ v
        nwv = math.sqrt(float(wv @ wv))
        if nwv == 0.0:
            raise ZeroDivisionError("power iteration hit W v = 0")
        u = wv / nwv
        w = W.T @ u
        sig = math.sqrt(float(w @ w))
        v = w / sig
    return W / sig, sig, v


def prescale_frobenius(W: np.ndarray):
    """W / |W|_F (R3: |W|_F >= sigma_max, always a safe start)."""
    W = np.asarray(W, dtype=np.float64)
    if W.size == 0:
        return W.copy(), 0.0
    f = math.sqrt(float(np.sum(W * W)))
    if f == 0.0:
        raise ZeroDivisionError("zero matrix (S:115)")
    return W / f, f


# ---------------------------------------------------------------------------
# O3: Bjorck-Bowie iteration (eq. P:308-312; R1, R4)
# ---------------------------------------------------------------------------
def bjorck(W0: np.ndarray, T: int, beta: float = 0.5) -> np.ndarray:
    """T iterations of W <- (1+beta) W - beta W W^T W.  The Gram is
    formed on the short side (associativity, R4): m >= n uses W (W^T W),
    m < n uses (W W^T) W."""
    W = np.asarray(W0, dtype=np.float64).copy()
    if W.size == 0:
        return W
    m, n = W.shape
    for _ in range(T):
        if m >= n:
            W = (1.0 + beta) * W - beta * (W @ (W.T @ W))
        else:
            W = (1.0 + beta) * W - beta * ((W @ W.T) @ W)
    return W


def ns_residual(X: np.ndarray) -> float:
    """|I - X^T X|_F on the short side (the NS residual)."""
    X = np.asarray(X, dtype=np.float64)
    if X.size == 0:
        return 0.0
    m, n = X.shape
    G = X.T @ X if m >= n else X @ X.T
    return float(np.linalg.norm(np.eye(G.shape[0]) - G))


def orthogonalize(mats: Sequence[np.ndarray], T: int = 12, beta: float = 0.5,
                  prescale: str = "power", P: int = 3,
                  v: Optional[Sequence[np.ndarray]] = None):
    """a2+a3 for a list of matrices: pre-scale then Bjorck.  v: one start
    vector per matrix (length n); None -> ones/sqrt(n) (R2).  Returns
    (ortho_list, v_new_list)."""
    outs, vs = [], []
    for idx, W in enumerate(mats):
        W = np.asarray(W, dtype=np.float64)
        n = W.shape[1]
        if W.size == 0:
            outs.append(W.copy())
            vs.append(np.zeros(n))
            continue
        if prescale == "power":
            v0 = np.ones(n) / math.sqrt(n) if v is None else np.asarray(v[idx], np.float64)
            W0, _, vn = prescale_power(W, P, v0)
        else:
            W0, _ = prescale_frobenius(W)
            vn = np.zeros(n) if v is None else np.asarray(v[idx], np.float64)
        outs.append(bjorck(W0, T, beta))
        vs.append(vn)
    return outs, vs


# ---------------------------------------------------------------------------
# O4-O7: block convolution and the AOC construction
# ---------------------------------------------------------------------------
def block_conv(K1: np.ndarray, K2: np.ndarray) -> np.ndarray:
    """K1 (*) K2: the kernel of conv_{K1} o conv_{K2} (P:351 footnote).
    K[:, :, a+c, b+e] += K1[:, :, a, b] @ K2[:, :, c, e]."""
    A, B, h1, w1 = K1.shape
    B2, C, h2, w2 = K2.shape
    if B != B2:
        raise ValueError("inner channel mismatch")
    K = np.zeros((A, C, h1 + h2 - 1, w1 + w2 - 1))
    for a in range(h1):
        for b in range(w1):
            for c in range(h2):
                for e in range(w2):
                    K[:, :, a + c, b + e] += K1[:, :, a, b] @ K2[:, :, c, e]
    return K


def block_orth(Pa: np.ndarray, Pb: np.ndarray) -> np.ndarray:
    """2x2 BCOP block [[PaPb, Pa(I-Pb)], [(I-Pa)Pb, (I-Pa)(I-Pb)]] (R5; the
    [P | I-P] elementary kernels of S:232 composed vertically then
    horizontally; "composing elementary orthogonal building blocks")."""
    c = Pa.shape[0]
    I = np.eye(c)
    K = np.zeros((c, c, 2, 2))
    K[:, :, 0, 0] = Pa @ Pb
    K[:, :, 0, 1] = Pa @ (I - Pb)
    K[:, :, 1, 0] = (I - Pa) @ Pb
    K[:, :, 1, 1] = (I - Pa) @ (I - Pb)
    return K


def bcop(Q: np.ndarray, Us: Sequence[np.ndarray], c_out: int, c_in: int) -> np.ndarray:
    """BCOP kernel (R5/R6): P_j = U_j U_j^T;
    K = Q (*) B_1 (*) ... (*) B_{k'-1}, B_j = block_orth(P_{2j-1}, P_{2j});
    sliced to [:c_out, :c_in]."""
    c = Q.shape[0]
    K = np.asarray(Q, np.float64)[:, :, None, None]
    Ps = [np.asarray(U, np.float64) @ np.asarray(U, np.float64).T if U.size else np.zeros((c, c))
          for U in Us]
    for j in range(len(Ps) // 2):
        K = block_conv(K, block_orth(Ps[2 * j], Ps[2 * j + 1]))
    return K[:c_out, :c_in]


def rko(R: np.ndarray, c_out: int, c_mid: int, s: int) -> np.ndarray:
    """RKO kernel: reshape of the semi-orthogonal R to (c_out, c_mid, s, s) in
    C order (R7)."""
    return np.asarray(R, np.float64).reshape(c_out, c_mid, s, s)


def layer_kernel(L: Layer, group_mats: Sequence[Sequence[np.ndarray]]) -> np.ndarray:
    """AOC kernel of one layer from its ORTHOGONALISED matrices, one list per
    group in layer_matrices() order (R7, R8, R13, R15).
    Returns the forward-conv kernel (co_f, ci_f/g, k, k); for 'dense' the
    co x ci matrix."""
    geo = layer_geometry(L)
    ks = []
    for mats in group_mats:
        mats = [np.asarray(M, np.float64) for M in mats]
        if geo["kind"] == "dense":
            ks.append(mats[0])
            continue
        if geo["kind"] == "soc":
            ks.append(soc_exp_kernel(mats[0].reshape(geo["co"], geo["ci"], L.k, L.k), L.terms)[0])
            continue
        if geo["kind"] == "sll":
            ks.append(aol_rescale(mats[0].reshape(geo["co"], geo["ci"], L.k, L.k)))
            continue
        if geo["kind"] == "bcop":
            ks.append(bcop(mats[0], mats[1:], geo["co"], geo["ci"]))
        elif geo["kind"] == "rko":
            ks.append(rko(mats[0], geo["co"], geo["ci"], L.s))
        else:
            Kb = bcop(mats[0], mats[1:-1], geo["c_mid"], geo["ci"])
            Kr = rko(mats[-1], geo["co"], geo["c_mid"], L.s)
            ks.append(block_conv(Kr, Kb))
    return np.concatenate(ks, axis=0)


# ---------------------------------------------------------------------------
# O8/O9: convolution and its adjoint
# ---------------------------------------------------------------------------
def out_size(H: int, k: int, s: int, d: int, p0: int, p1: int) -> int:
    """H_out = floor((H + p0 + p1 - d(k-1) - 1)/s) + 1."""
    return (H + p0 + p1 - d * (k - 1) - 1) // s + 1


def _tap_rows(H: int, Ho: int, s: int, d: int, a: int, p0: int, circular: bool):
    r = s * np.arange(Ho) + d * a - p0
    if circular:
        return np.mod(r, H), np.ones(Ho, bool)
    ok = (r >= 0) & (r < H)
    return np.clip(r, 0, H - 1), ok


def conv2d(x: np.ndarray, K: np.ndarray, s: int = 1, d: int = 1, g: int = 1,
           pads=None, mode: str = "circular") -> np.ndarray:
    """Strided/dilated/grouped cross-correlation (a6):
    y[n,o,u,v] = sum_{i in grp(o)} sum_{a,b} K[o,i,a,b] x~[n, i, s u + d a - p_t, s v + d b - p_l],
    x~ zero-extended or circular (index mod H).  Direct tap loops with a
    channel matmul per tap."""
    x = np.asarray(x, np.float64)
    K = np.asarray(K, np.float64)
    N, C, H, W = x.shape
    Co, Cig, kh, kw = K.shape
    if C != Cig * g or Co % g:
        raise ValueError("channel/group mismatch")
    if pads is None:
        e = d * (kh - 1)
        pads = (e // 2, e - e // 2, e // 2, e - e // 2)
    pt, pb, pl, pr = pads
    Ho, Wo = out_size(H, kh, s, d, pt, pb), out_size(W, kw, s, d, pl, pr)
    circ = mode == "circular"
    Cog = Co // g
    y = np.zeros((N, Co, Ho, Wo))
    for a in range(kh):
        rows, rok = _tap_rows(H, Ho, s, d, a, pt, circ)
        for b in range(kw):
            cols, cok = _tap_rows(W, Wo, s, d, b, pl, circ)
            patch = x[:, :, rows][:, :, :, cols] * (rok[:, None] & cok[None, :])
            for gi in range(g):
                xs = patch[:, gi * Cig:(gi + 1) * Cig]
                Kt = K[gi * Cog:(gi + 1) * Cog, :, a, b]
                y[:, gi * Cog:(gi + 1) * Cog] += np.einsum("oi,nihw->nohw", Kt, xs)
    return y


def conv_transpose2d(y: np.ndarray, K: np.ndarray, H: int, W: int, s: int = 1,
                     d: int = 1, g: int = 1, pads=None, mode: str = "circular") -> np.ndarray:
    """Exact adjoint of conv2d(., K, spec) on (H, W) inputs (a7, R13,
    R14): scatter form x~[n, i, s u + d a - p_t, s v + d b - p_l] += K[o,i,a,b] y[n,o,u,v],
    wrapped mod H (circular) or dropped when out of range (zeros)."""
    y = np.asarray(y, np.float64)
    K = np.asarray(K, np.float64)
    N, Co, Ho, Wo = y.shape
    _, Cig, kh, kw = K.shape
    if pads is None:
        e = d * (kh - 1)
        pads = (e // 2, e - e // 2, e // 2, e - e // 2)
    pt, pb, pl, pr = pads
    if (Ho, Wo) != (out_size(H, kh, s, d, pt, pb), out_size(W, kw, s, d, pl, pr)):
        raise ValueError("shape mismatch")
    circ = mode == "circular"
    Cog = Co // g
    x = np.zeros((N, Cig * g, H, W))
    for a in range(kh):
        rows, rok = _tap_rows(H, Ho, s, d, a, pt, circ)
        for b in range(kw):
            cols, cok = _tap_rows(W, Wo, s, d, b, pl, circ)
            mask = (rok[:, None] & cok[None, :])
            for gi in range(g):
                Kt = K[gi * Cog:(gi + 1) * Cog, :, a, b]
                contrib = np.einsum("oi,nohw->nihw", Kt, y[:, gi * Cog:(gi + 1) * Cog]) * mask
                # unbuffered scatter-add: repeated (wrapped) targets accumulate
                np.add.at(x, (slice(None), slice(gi * Cig, (gi + 1) * Cig),
                              rows[:, None], cols[None, :]), contrib)
    return x


# ---------------------------------------------------------------------------
# O10: verifiers
# ---------------------------------------------------------------------------
def toeplitz(op, in_shape: Tuple[int, int, int]) -> np.ndarray:
    """Matrix of a linear op by impulse responses ("Using the impulse
    response approach, we construct the Toeplitz matrix"): column j =
    flatten(op(e_j))."""
    C, H, W = in_shape
    n = C * H * W
    E = np.eye(n).reshape(n, C, H, W)
    Y = op(E)
    return Y.reshape(n, -1).T


def fft_singular_values(K: np.ndarray, H: int, W: int, d: int = 1) -> np.ndarray:
    """Singular values of the circular stride-1 conv on H x W by per-frequency
    SVD (P:433 FFT lineage).  Transfer matrix at (f1, f2):
    M = sum_{a,b} K[:, :, a, b] exp(2 pi i (f1 d a / H + f2 d b / W))."""
    Co, Ci, kh, kw = K.shape
    out = []
    for f1 in range(H):
        for f2 in range(W):
            M = np.zeros((Co, Ci), complex)
            for a in range(kh):
                for b in range(kw):
                    M += K[:, :, a, b] * np.exp(2j * np.pi * (f1 * d * a / H + f2 * d * b / W))
            out.append(np.linalg.svd(M, compute_uv=False))
    return np.sort(np.concatenate(out))


def polyphase_singular_values(K: np.ndarray, H: int, W: int, s: int, d: int = 1,
                              pads=None) -> np.ndarray:
    """Singular values of the circular stride-s conv (s | H, s | W) via the
    polyphase reduction: with t = d a - p = s q + r,
    x[s u + t] = x_r[u + q], so the strided conv is a stride-1 conv on the
    s^2-phase input; per-frequency SVD of the c_out x (c_in s^2) symbol on the
    (H/s) x (W/s) grid."""
    Co, Ci, kh, kw = K.shape
    if H % s or W % s:
        raise ValueError("polyphase needs s | H and s | W")
    if pads is None:
        e = d * (kh - 1)
        pads = (e // 2, e - e // 2, e // 2, e - e // 2)
    pt, _, pl, _ = pads
    Hs, Ws = H // s, W // s
    out = []
    for f1 in range(Hs):
        for f2 in range(Ws):
            M = np.zeros((Co, Ci, s, s), complex)
            for a in range(kh):
                qa, ra = divmod(d * a - pt, s)
                for b in range(kw):
                    qb, rb = divmod(d * b - pl, s)
                    M[:, :, ra, rb] += K[:, :, a, b] * np.exp(2j * np.pi * (f1 * qa / Hs + f2 * qb / Ws))
            out.append(np.linalg.svd(M.reshape(Co, Ci * s * s), compute_uv=False))
    return np.sort(np.concatenate(out))


def conv_singular_values(K: np.ndarray, L: Layer, H: int, W: int) -> np.ndarray:
    """All singular values of a circular layer operator on H x W inputs,
    group by group (block-diagonal), using FFT (s = 1) or polyphase."""
    g = L.g
    Cog = K.shape[0] // g
    vals = []
    for gi in range(g):
        Kg = K[gi * Cog:(gi + 1) * Cog]
        if L.s == 1:
            vals.append(fft_singular_values(Kg, H, W, L.d))
        else:
            vals.append(polyphase_singular_values(Kg, H, W, L.s, L.d, L.pads()))
    return np.sort(np.concatenate(vals))


def spectral_certificate(K: np.ndarray, L: Layer, H: int, W: int):
    """Per (group, frequency) spectral certificate of the circular layer operator on H x W (SURVEY §8(f)
    row 2; App. C "scalable spectral norm estimation ... check that the produced bounds are
    valid"; S:444-452 fft_circular_spectrum).

    For each group and each frequency (f1, f2) of the (H/s) x (W/s) polyphase grid it forms the symbol M
    exactly as polyphase_singular_values does (c_out/g x (c_in/g) s^2, complex), the Gram on the SHORT
    side G = M^H M (or M M^H), E = G - I, and returns
      frob[g, f1, f2]   = |E|_F            (certificate: max |sigma^2 - 1| <= |E|_2 <= |E|_F, and
                                            |sigma - 1| <= |sigma^2 - 1| for sigma >= 0),
      spec[g, f1, f2]   = |E|_2            (eigvalsh: = max |sigma^2 - 1| at that frequency),
      sigma_dev         = max over everything of |sigma - 1| (np.linalg.svd of M).
    Dense layers: one 'frequency', M = the kernel matrix."""
    if L.kind == "dense":
        K = K.reshape(K.shape[0], K.shape[1], 1, 1)
        s, d, pt, pl, H, W = 1, 1, 0, 0, 1, 1
    else:
        s, d = L.s, L.d
        pt, _, pl, _ = L.pads()
    if H % s or W % s:
        raise ValueError("certificate needs s | H and s | W")
    Co, Ci, kh, kw = K.shape
    g = 1 if L.kind == "dense" else L.g
    Cog = Co // g
    Hs, Ws = H // s, W // s
    frob = np.zeros((g, Hs, Ws))
    spec = np.zeros((g, Hs, Ws))
    sig_dev = 0.0
    for gi in range(g):
        Kg = K[gi * Cog:(gi + 1) * Cog]
        for f1 in range(Hs):
            for f2 in range(Ws):
                M = np.zeros((Cog, Ci, s, s), complex)
                for a in range(kh):
                    qa, ra = divmod(d * a - pt, s)
                    for b in range(kw):
                        qb, rb = divmod(d * b - pl, s)
                        M[:, :, ra, rb] += Kg[:, :, a, b] * np.exp(2j * np.pi * (f1 * qa / Hs + f2 * qb / Ws))
                M = M.reshape(Cog, Ci * s * s)
                G = M.conj().T @ M if M.shape[0] >= M.shape[1] else M @ M.conj().T
                E = G - np.eye(G.shape[0])
                frob[gi, f1, f2] = np.linalg.norm(E)
                spec[gi, f1, f2] = np.abs(np.linalg.eigvalsh(E)).max()
                sig_dev = max(sig_dev, float(np.abs(np.linalg.svd(M, compute_uv=False) - 1).max()))
    return frob, spec, sig_dev


# ---------------------------------------------------------------------------
# f3: Adaptive-SOC explicit exponential (§3 "Adaptive-SOC"; P:349-361
# App. B.2 Theorem "Explicit conv exponential"; readings R25-R27)
# ---------------------------------------------------------------------------
def soc_skew(K: np.ndarray) -> np.ndarray:
    """Skew-symmetrised free kernel (S:262 step 1): L[a, b, i, j] = (K[a, b, i, j] - K[b, a, k-1-i, k-1-j]) / 2.
    With centred padding (odd k) the circular operator of L is skew-adjoint: T(L)^T = -T(L)."""
    K = np.asarray(K, np.float64)
    return 0.5 * (K - np.transpose(K, (1, 0, 2, 3))[:, :, ::-1, ::-1])


def aol_scale(L: np.ndarray) -> float:
    """Scalar AOL normalisation (S:262 step 2, "We used 'AOL'", S:269-276 aol_rescale; reading R26):
    V[i, j, Delta] = sum_o sum_t L[o, i, t] L[o, j, t + Delta] (the full cross-correlation of the kernel with
    itself, contracted over output channels), d_i = sum_j sum_Delta |V[i, j, Delta]|.  AOL: |T D^{-1/2}| <= 1,
    hence |T(L)| <= max_i sqrt(d_i); the returned alpha = 1 / max_i sqrt(d_i) gives |T(alpha L)| <= 1 while
    keeping alpha L skew (a per-channel rescale would not).  d = 0 (L = 0) -> alpha = 1."""
    L = np.asarray(L, np.float64)
    co, ci, k1, k2 = L.shape
    d = np.zeros(ci)
    for da in range(-(k1 - 1), k1):
        for db in range(-(k2 - 1), k2):
            V = np.zeros((ci, ci))
            for a in range(k1):
                for b in range(k2):
                    a2, b2 = a + da, b + db
                    if 0 <= a2 < k1 and 0 <= b2 < k2:
                        V += L[:, :, a, b].T @ L[:, :, a2, b2]
            d += np.abs(V).sum(axis=1)
    m = float(np.sqrt(d.max()))
    return 1.0 / m if m > 0 else 1.0


def soc_exp_kernel(K: np.ndarray, terms: int):
    """Explicit exponential kernel (eq. "(Id + K + K(*)K/2! + K(*)K(*)K/3! + ...) * x"):
    L = alpha soc_skew(K) (alpha = aol_scale), E = delta + sum_{j=1..terms} L^{(*) j} / j!, every term centred
    in the (terms (k-1) + 1)^2 output (odd k: "same" padding composes by adding the pads).  Returns (E, alpha)."""
    K = np.asarray(K, np.float64)
    c, c2, k, k2 = K.shape
    if c != c2 or k != k2 or k % 2 == 0:
        raise ValueError("SOC needs a square channel map and an odd square kernel")
    Ls = soc_skew(K)
    alpha = aol_scale(Ls)
    L = alpha * Ls
    kn = terms * (k - 1) + 1
    E = np.zeros((c, c, kn, kn))
    ctr = (kn - 1) // 2
    E[:, :, ctr, ctr] = np.eye(c)
    P = np.eye(c)[:, :, None, None]
    fact = 1.0
    for j in range(1, terms + 1):
        P = block_conv(P, L)
        fact *= j
        off = (terms - j) * (k - 1) // 2
        kj = P.shape[2]
        E[:, :, off:off + kj, off:off + kj] += P / fact
    return E, alpha


# ---------------------------------------------------------------------------
# f4: SLL x AOC fused down-sampling block (App. B.3; readings R28-R30)
# ---------------------------------------------------------------------------
def aol_rescale(K: np.ndarray) -> np.ndarray:
    """AOL per-input-channel rescale (P:133 AOL; the SLL kernel K = W T^{-1/2} of P:389 with the
    SDP scaling q = 1, reading R28): V[i, j, Delta] = sum_o sum_t K[o, i, t] K[o, j, t + Delta],
    d_i = sum_j sum_Delta |V[i, j, Delta]|, input channel i scaled by d_i^{-1/2} (d_i = 0: unscaled).
    Then |T(K D^{-1/2})| <= 1 (Prach & Lampert)."""
    K = np.asarray(K, np.float64)
    co, ci, k1, k2 = K.shape
    d = np.zeros(ci)
    for da in range(-(k1 - 1), k1):
        for db in range(-(k2 - 1), k2):
            V = np.zeros((ci, ci))
            for a in range(k1):
                for b in range(k2):
                    a2, b2 = a + da, b + db
                    if 0 <= a2 < k1 and 0 <= b2 < k2:
                        V += K[:, :, a, b].T @ K[:, :, a2, b2]
            d += np.abs(V).sum(axis=1)
    sc = np.where(d > 0, 1.0 / np.sqrt(np.where(d > 0, d, 1.0)), 1.0)
    return K * sc[None, :, None, None]


def adjoint_kernel(K: np.ndarray) -> np.ndarray:
    """Kernel of the adjoint of a stride-1 conv: channels transposed, taps flipped (with the padding
    p -> k - 1 - p, see sll_block_kernels)."""
    return np.ascontiguousarray(np.transpose(np.asarray(K, np.float64), (1, 0, 2, 3))[:, :, ::-1, ::-1])


def same_pads(k: int, d: int = 1):
    """Reading R11: p_t = floor(d(k-1)/2), p_b = d(k-1) - p_t (same on both axes)."""
    e = d * (k - 1)
    return (e // 2, e - e // 2, e // 2, e - e // 2)


def sll_block_kernels(K_pre: np.ndarray, K_post: np.ndarray, W_sll: np.ndarray):
    """The block's merged kernels ("kernels are merged once per batch"):
    K = aol_rescale(W_sll);  C = K (*) K_pre;  A = K_post (*) K_pre;  B = K_post (*) adjoint(K).
    Padding of a composition is the sum of the factors' (top/left) pads; the adjoint of a "same" conv with
    top pad p has top pad k - 1 - p.  A and B are merged into ONE kernel over the concatenated input
    [x | h]: M = [A | -2 B], each embedded at offset P - p in a common window with top pad P = max(pA, pB)
    (reading R29).  Returns dict(C, padC, M, padM, K, A, B)."""
    K = aol_rescale(W_sll)
    kpre, kpost, ks = K_pre.shape[2], K_post.shape[2], K.shape[2]
    ppre, ppost, ps = same_pads(kpre)[0], same_pads(kpost)[0], same_pads(ks)[0]
    C = block_conv(K, K_pre)
    A = block_conv(K_post, K_pre)
    B = block_conv(K_post, adjoint_kernel(K))
    pC, pA, pB = ps + ppre, ppost + ppre, ppost + (ks - 1 - ps)
    P = max(pA, pB)
    kM = max(P - pA + A.shape[2], P - pB + B.shape[2])
    co, c, cs = A.shape[0], A.shape[1], B.shape[1]
    M = np.zeros((co, c + cs, kM, kM))
    oa, ob = P - pA, P - pB
    M[:, :c, oa:oa + A.shape[2], oa:oa + A.shape[3]] = A
    M[:, c:, ob:ob + B.shape[2], ob:ob + B.shape[3]] = -2.0 * B
    kC = C.shape[2]
    return dict(C=C, padC=(pC, kC - 1 - pC, pC, kC - 1 - pC), M=M, padM=(P, kM - 1 - P, P, kM - 1 - P),
                K=K, A=A, B=B)


def sll_block_forward(x: np.ndarray, kern: dict, b: np.ndarray, s: int) -> np.ndarray:
    """Fused block: y = M *_s [x | relu(C * x + b)], circular (reading R30)."""
    h = conv2d(x, kern["C"], pads=kern["padC"]) + np.asarray(b, np.float64)[None, :, None, None]
    z = np.concatenate([np.asarray(x, np.float64), np.maximum(h, 0.0)], axis=1)
    return conv2d(z, kern["M"], s=s, pads=kern["padM"])


def sll_block_unfused(x: np.ndarray, K_pre: np.ndarray, K_post: np.ndarray, K: np.ndarray, b: np.ndarray,
                      s: int) -> np.ndarray:
    """The block as three sequential layers: z = K_pre * x; u = z - 2 K^T * relu(K * z + b)
    (SLL; K^T * = the exact adjoint conv); y = K_post *_s u.  Circular, "same" pads."""
    z = conv2d(x, K_pre)
    t = np.maximum(conv2d(z, K) + np.asarray(b, np.float64)[None, :, None, None], 0.0)
    u = z - 2.0 * conv_transpose2d(t, K, z.shape[2], z.shape[3])
    return conv2d(u, K_post, s=s)


# ---------------------------------------------------------------------------
# f1: backward of the path ("per-batch cost grows as soon as weights are
# iteratively projected", P:122 the <= 1.13x ImageNet TRAINING wall time; readings R31-R33)
# ---------------------------------------------------------------------------
def conv2d_wgrad(x: np.ndarray, dy: np.ndarray, kshape, s: int = 1, d: int = 1, g: int = 1, pads=None,
                 mode: str = "circular") -> np.ndarray:
    """Weight gradient of conv2d (the bilinear form <dy, conv2d(x, dK)> = <wgrad, dK>):
    dK[o, i, a, b] = sum_{n,u,v} dy[n, o, u, v] x~[n, grp(o) i, s u + d a - p_t, s v + d b - p_l]."""
    x = np.asarray(x, np.float64)
    dy = np.asarray(dy, np.float64)
    N, C, H, W = x.shape
    Co, Cig, kh, kw = kshape
    if pads is None:
        pads = same_pads(kh, d)
    pt, pb, pl, pr = pads
    Ho, Wo = dy.shape[2], dy.shape[3]
    circ = mode == "circular"
    Cog = Co // g
    dK = np.zeros(kshape)
    for a in range(kh):
        rows, rok = _tap_rows(H, Ho, s, d, a, pt, circ)
        for b in range(kw):
            cols, cok = _tap_rows(W, Wo, s, d, b, pl, circ)
            patch = x[:, :, rows][:, :, :, cols] * (rok[:, None] & cok[None, :])
            for gi in range(g):
                dK[gi * Cog:(gi + 1) * Cog, :, a, b] = np.einsum(
                    "nohw,nihw->oi", dy[:, gi * Cog:(gi + 1) * Cog], patch[:, gi * Cig:(gi + 1) * Cig])
    return dK


def bjorck_vjp(W0: np.ndarray, T: int, beta: float, G: np.ndarray) -> np.ndarray:
    """VJP of bjorck(W0, T, beta) (the forward iteration of O3, replayed): with A = X^T X, the step
    X' = (1+beta) X - beta X A has the adjoint dX = (1+beta) G - beta (G A + X G^T X + X X^T G)  (m >= n;
    for m < n the transposed form).  Iterates are recomputed, then reversed."""
    X = np.asarray(W0, np.float64)
    m, n = X.shape
    xs = []
    for _ in range(T):
        xs.append(X)
        X = (1 + beta) * X - beta * (X @ (X.T @ X) if m >= n else (X @ X.T) @ X)
    G = np.asarray(G, np.float64)
    for X in reversed(xs):
        if m >= n:
            G = (1 + beta) * G - beta * (G @ (X.T @ X) + X @ G.T @ X + X @ X.T @ G)
        else:
            G = (1 + beta) * G - beta * ((X @ X.T) @ G + X @ G.T @ X + G @ X.T @ X)
    return G


def orthogonalize_vjp(mats, G, T: int = 12, beta: float = 0.5, prescale: str = "power", P: int = 3, v=None):
    """VJP of orthogonalize (a2 + a3) with the pre-scale treated as a constant (reading R31: sigma is a
    stop-gradient preconditioner; at convergence the polar factor is scale-invariant so its derivative along
    W is 0 anyway): dW = bjorck_vjp(W / sigma, T, beta, G) / sigma."""
    out = []
    for idx, W in enumerate(mats):
        W = np.asarray(W, np.float64)
        if W.size == 0:
            out.append(W.copy())
            continue
        n = W.shape[1]
        if prescale == "power":
            v0 = np.ones(n) / math.sqrt(n) if v is None else np.asarray(v[idx], np.float64)
            W0, sig, _ = prescale_power(W, P, v0)
        else:
            W0, sig = prescale_frobenius(W)
        out.append(bjorck_vjp(W0, T, beta, G[idx]) / sig)
    return out


def block_conv_vjp(K1: np.ndarray, K2: np.ndarray, dK: np.ndarray):
    """Adjoint of block_conv in both factors: dK1[a] = sum_c dK[a + c] K2[c]^T, dK2[c] = sum_a K1[a]^T dK[a + c]."""
    _, _, h1, w1 = K1.shape
    _, _, h2, w2 = K2.shape
    d1, d2 = np.zeros(K1.shape), np.zeros(K2.shape)
    for a in range(h1):
        for b in range(w1):
            for c in range(h2):
                for e in range(w2):
                    d1[:, :, a, b] += dK[:, :, a + c, b + e] @ K2[:, :, c, e].T
                    d2[:, :, c, e] += K1[:, :, a, b].T @ dK[:, :, a + c, b + e]
    return d1, d2


def _bcop_vjp(Q, Us, c_out, c_in, dK):
    c = Q.shape[0]
    I = np.eye(c)
    Ps = [np.asarray(U, np.float64) @ np.asarray(U, np.float64).T if U.size else np.zeros((c, c)) for U in Us]
    Ks = [np.asarray(Q, np.float64)[:, :, None, None]]
    Bs = []
    for j in range(len(Ps) // 2):
        Bs.append(block_orth(Ps[2 * j], Ps[2 * j + 1]))
        Ks.append(block_conv(Ks[-1], Bs[-1]))
    dcur = np.zeros(Ks[-1].shape)
    dcur[:c_out, :c_in] = dK                                # adjoint of the slice: zero padding
    dPs = [None] * len(Ps)
    for j in reversed(range(len(Bs))):
        dprev, dB = block_conv_vjp(Ks[j], Bs[j], dcur)
        Pa, Pb = Ps[2 * j], Ps[2 * j + 1]
        d00, d01, d10, d11 = dB[:, :, 0, 0], dB[:, :, 0, 1], dB[:, :, 1, 0], dB[:, :, 1, 1]
        dPs[2 * j] = d00 @ Pb.T + d01 @ (I - Pb).T - d10 @ Pb.T - d11 @ (I - Pb).T
        dPs[2 * j + 1] = Pa.T @ d00 - Pa.T @ d01 + (I - Pa).T @ d10 - (I - Pa).T @ d11
        dcur = dprev
    dQ = dcur[:, :, 0, 0]
    dUs = [(dP + dP.T) @ np.asarray(U, np.float64) if U.size else np.zeros(U.shape) for dP, U in zip(dPs, Us)]
    return [dQ] + dUs


def layer_kernel_vjp(L: Layer, group_mats, dK: np.ndarray):
    """Adjoint of layer_kernel (a4 + a5) for AOC / BCOP / RKO / dense layers: per group the matrix gradients
    in layer_matrices() order, from the gradient of the forward-conv kernel (co_f, ci_f/g, k, k)."""
    geo = layer_geometry(L)
    co = geo["co"]
    out = []
    for gi, mats in enumerate(group_mats):
        mats = [np.asarray(M, np.float64) for M in mats]
        dKg = np.asarray(dK, np.float64)[gi * co:(gi + 1) * co]
        if geo["kind"] == "dense":
            out.append([dKg.reshape(mats[0].shape)])
        elif geo["kind"] == "bcop":
            out.append(_bcop_vjp(mats[0], mats[1:], geo["co"], geo["ci"], dKg))
        elif geo["kind"] == "rko":
            out.append([dKg.reshape(mats[0].shape)])
        elif geo["kind"] == "aoc":
            Kb = bcop(mats[0], mats[1:-1], geo["c_mid"], geo["ci"])
            Kr = rko(mats[-1], geo["co"], geo["c_mid"], L.s)
            dKr, dKb = block_conv_vjp(Kr, Kb, dKg)
            out.append(_bcop_vjp(mats[0], mats[1:-1], geo["c_mid"], geo["ci"], dKb) + [dKr.reshape(mats[-1].shape)])
        else:
            raise ValueError(f"no VJP for {geo['kind']}")
    return out
