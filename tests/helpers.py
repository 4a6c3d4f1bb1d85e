"""Shared test helpers: seeded packing of parameters (synth) and the oracle
construction of the same inputs.  The oracle never sees a value produced by
the CUDA path; GPU outputs are only ever compared against it or checked by
its verifiers."""
from __future__ import annotations

import numpy as np

import oracle as O
from synth import gen


def oracle_layer(d) -> O.Layer:
    return O.Layer(d["c_in"], d["c_out"], d.get("k", 3), d.get("s", 1), d.get("d", 1), d.get("g", 1),
                   kind=d.get("kind", "conv"), padding_mode=d.get("padding_mode", "circular"),
                   pad=d.get("pad"), terms=d.get("terms", 6) or 6)


def pack_params(plan, cfg_id: int, stress: bool = False):
    """float32 flat params buffer in the plan's layout + the list of matrices."""
    buf = np.zeros(plan.params_numel, np.float32)
    mats = []
    for i, m in enumerate(plan.matrices):
        A = gen.param_matrix(m["m"], m["n"], (cfg_id, m["layer"], m["group"], i, gen.ROLE_ID[m["role"]]), stress)
        buf[m["off"]: m["off"] + A.size] = A.ravel()
        mats.append(A)
    return buf, mats


def pack_cache(plan, cfg_id: int):
    buf = np.zeros(plan.cache_numel, np.float32)
    vs = []
    for i, m in enumerate(plan.matrices):
        v = gen.unit_vector(m["n"], (cfg_id, m["layer"], m["group"], i, gen.ROLE_ID["v"]))
        buf[m["cache_off"]: m["cache_off"] + v.size] = v
        vs.append(v)
    return buf, vs


def oracle_construct(layers, mats, T=12, beta=0.5, prescale="power", P=3, v=None):
    """Oracle a2..a5 on the float32 matrices (upcast to f64).  SOC free kernels (role K) are not
    orthogonalised (f3): they pass through to the explicit exponential."""
    roles = [M.role for d in layers for _ in range(d.get("g", 1) if d.get("kind") != "dense" else 1)
             for M in O.layer_matrices(oracle_layer(d))]
    ortho, vnew = O.orthogonalize([A.astype(np.float64) for A in mats], T=T, beta=beta, prescale=prescale, P=P,
                                  v=None if v is None else [x.astype(np.float64) for x in v])
    ortho = [A.astype(np.float64) if r == "K" else X for A, X, r in zip(mats, ortho, roles)]
    kernels, idx = [], 0
    for d in layers:
        OL = oracle_layer(d)
        if d.get("kind") == "sll_block":   # f4: merged from three earlier layers' kernels -> (C, M) dict
            kernels.append(O.sll_block_kernels(kernels[d["pre"]], kernels[d["post"]],
                                               sll_free_kernel(layers, d["sll"], ortho)))
            continue
        nm = len(O.layer_matrices(OL))
        groups = []
        for _ in range(OL.g):
            groups.append(ortho[idx: idx + nm])
            idx += nm
        kernels.append(O.layer_kernel(OL, groups))
    return ortho, vnew, kernels


def sll_free_kernel(layers, l, mats):
    """The free (not yet AOL-rescaled) kernel of SLL layer l from the packed matrix list."""
    idx = 0
    for j, d in enumerate(layers):
        nm = len(O.layer_matrices(oracle_layer(d))) * (d.get("g", 1) if d.get("kind") != "dense" else 1)
        if j == l:
            W = np.asarray(mats[idx], np.float64)
            return W.reshape(d["c_out"], d["c_in"], d.get("k", 3), d.get("k", 3))
        idx += nm
    raise IndexError(l)


def rel(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def nchw(x_nhwc):
    return np.ascontiguousarray(np.transpose(x_nhwc, (0, 3, 1, 2)))


def nhwc(x_nchw):
    return np.ascontiguousarray(np.transpose(x_nchw, (0, 2, 3, 1)))


# Elementwise bounds of a conv output, on top of the Frobenius ratio:
#   |gpu - ref| <= rel * |ref| + coef * (|K| * |x|)
# where (|K| * |x|) is the oracle conv of the absolute values (the tap-sum of |K||x| of every output
# element).  BF16 I/O with the same BF16 kernel on both sides: the products are exact in FP32, so the
# error is the output RNE rounding (<= 2^-8 |y|) plus the FP32 accumulation (<< 2^-12 of the tap-sum).
BF16_ELEM = (2.0 ** -8, 2.0 ** -12)
F32_ELEM = (2.0 ** -20, 2.0 ** -16)


def assert_elementwise(got, ref, absref, rel_coef, abs_coef, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref)
    bound = rel_coef * np.abs(ref) + abs_coef * np.asarray(absref, np.float64) + 1e-30
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err / bound), err.shape)
        raise AssertionError(f"{what}: {int(bad.sum())} of {err.size} elements outside the bound; worst at {i}: "
                             f"got {got[i]:.6g} ref {ref[i]:.6g} bound {bound[i]:.3g}")
