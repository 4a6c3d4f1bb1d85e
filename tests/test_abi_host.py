"""Host-side tests of the C-ABI library (no GPU): symbol exports, validation
and rejection rules, unit derivation against the oracle, packed layouts,
construction sharding (LPT, rank-major segments) and the no-device contract."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2601_13776_b200 as orth
from synth import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "orth.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(orth_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = _declared_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(orth._lib, s), s
    assert set(syms) == set(orth.EXPORTED)


def L(**kw):
    d = dict(kind="conv", c_in=8, c_out=8, k=3, s=1, d=1, g=1, padding_mode="circular")
    d.update(kw)
    return d


@pytest.mark.parametrize("layer,status", [
    (L(), orth.OK),
    (L(g=3), orth.INVALID_ARGUMENT),                 # g must divide channels
    (L(c_in=0), orth.INVALID_ARGUMENT),              # dims >= 1
    (L(k=1, s=2), orth.UNSUPPORTED_CONFIG),          # k < s
    (L(s=2, d=2), orth.UNSUPPORTED_CONFIG),          # gcd(s, d) != 1 (R10)
    (L(s=2, d=4, k=3), orth.UNSUPPORTED_CONFIG),
    (L(s=2, d=3), orth.OK),                          # gcd = 1 accepted
    (L(c_in=1, c_out=8, s=2), orth.OK),              # c_out > c_in s^2 accepted (R9)
    (L(kind="dense", k=1), orth.OK),
    (L(kind="dense", k=3), orth.INVALID_ARGUMENT),
    (L(pad=(1, 1, 1, -1)), orth.INVALID_ARGUMENT),
    (L(kind="convT", padding_mode="circular", s=2), orth.OK),   # R14
])
def test_validation(layer, status):
    assert orth.orth_validate_desc([layer]) == status


@pytest.mark.parametrize("opts,status", [
    (dict(beta=0.0), orth.INVALID_ARGUMENT), (dict(beta=0.6), orth.INVALID_ARGUMENT),
    (dict(ns_iters=0), orth.INVALID_ARGUMENT), (dict(power_iters=0), orth.INVALID_ARGUMENT),
    (dict(rank=2, world=2), orth.INVALID_ARGUMENT), (dict(beta=0.25, ns_iters=30), orth.OK),
])
def test_validation_opts(opts, status):
    assert orth.orth_validate_desc([L()], **opts) == status


def test_create_raises_with_detail():
    with pytest.raises(orth.OrthError) as ei:
        orth.Plan([L(k=1, s=2)], device=-1)
    assert ei.value.status == orth.UNSUPPORTED_CONFIG
    assert "P:330" in str(ei.value)


def _oracle_layer(d):
    return O.Layer(d["c_in"], d["c_out"], d["k"], d["s"], d["d"], d["g"], kind=d["kind"],
                   padding_mode=d["padding_mode"])


GRID = [L(c_in=ci, c_out=co, k=k, s=s, d=dd, g=g, kind=kind)
        for (ci, co, k, s, dd, g, kind) in [
            (16, 16, 3, 1, 1, 1, "conv"), (4, 8, 3, 2, 1, 1, "conv"), (8, 4, 3, 2, 1, 1, "conv"),
            (1, 8, 3, 2, 1, 1, "conv"), (4, 16, 2, 2, 1, 1, "conv"), (8, 8, 4, 2, 1, 1, "conv"),
            (1, 1, 3, 1, 1, 1, "conv"), (8, 16, 3, 2, 1, 2, "conv"), (8, 8, 3, 1, 2, 2, "convT"),
            (4, 8, 3, 2, 1, 2, "convT"), (6, 9, 5, 3, 2, 3, "conv"), (3, 64, 4, 4, 1, 1, "conv")]]


@pytest.mark.parametrize("cfg", [configs.cfg1(), configs.cfg2(), configs.cfg3(), configs.cfg4(), GRID,
                                 configs.cfg5(512)[:4]])
def test_derivation_matches_oracle(cfg):
    p = orth.Plan(cfg, device=-1)
    mats = p.matrices
    idx = 0
    for l, d in enumerate(cfg):
        OL = _oracle_layer(d)
        spec = O.layer_matrices(OL)
        geo = O.layer_geometry(OL)
        info = p.layer_info[l]
        assert info["first_matrix"] == idx and info["mats_per_group"] == len(spec)
        assert info["c_mid"] == geo["c_mid"] and info["c_b"] == geo["c_b"] and info["kp"] == geo["kp"]
        for g in range(d["g"]):
            for j, M in enumerate(spec):
                m = mats[idx]
                assert (m["m"], m["n"], m["role"], m["layer"], m["group"]) == (M.m, M.n, M.role, l, g)
                idx += 1
        assert info["numel"] == int(np.prod(p.kernel_shape(l)))
    assert idx == p.n_matrices


def test_layout_alignment_and_disjointness():
    p = orth.Plan(configs.cfg2(), device=-1)
    end = 0
    for m in p.matrices:
        assert m["off"] % 32 == 0 and m["cache_off"] % 32 == 0
        assert m["off"] >= end
        end = m["off"] + m["m"] * m["n"]
    assert end <= p.params_numel
    ends = 0
    for l, info in enumerate(p.layer_info):
        assert info["kf32_off"] % 32 == 0 and info["kbf16_off"] % 64 == 0
        assert info["kf32_off"] >= ends
        ends = info["kf32_off"] + info["numel"]
    assert ends <= p.kf32_numel


@pytest.mark.parametrize("cfg_name", ["cfg3", "cfg4"])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_lpt_sharding_units_and_segments(cfg_name, world):
    """the sharding unit is (layer, group); LPT by NS flops (+ composition); every rank
    derives the same owners and offsets; each unit lies inside its owner's rank-major gather segment;
    the final layout is the single-rank one."""
    cfg = getattr(configs, cfg_name)()
    plans = [orth.Plan(cfg, device=-1, rank=r, world=world) for r in range(world)]
    single = orth.Plan(cfg, device=-1)
    units = plans[0].units
    assert [(u["layer"], u["group"]) for u in units] == [(l, g) for l, d in enumerate(cfg) for g in range(d["g"])]
    for p in plans[1:]:
        assert p.units == units
    seg = plans[0].seg_f32
    assert plans[0].gf32_numel == seg * world
    spans = sorted((u["gat_f32"], u["gat_f32"] + u["numel"]) for u in units)
    assert all(a1 <= b0 for (_, a1), (b0, _) in zip(spans, spans[1:]))          # disjoint
    for u in units:
        r = u["owner"]
        assert u["gat_f32"] % 32 == 0 and u["gat_bf16"] % 64 == 0
        assert r * seg <= u["gat_f32"] and u["gat_f32"] + u["numel"] <= (r + 1) * seg
        info = single.layer_info[u["layer"]]
        assert u["fin_f32"] == info["kf32_off"] + u["group"] * u["numel"]
        assert u["numel"] * cfg[u["layer"]]["g"] == info["numel"]
    assert [i["kf32_off"] for i in plans[0].layer_info] == [i["kf32_off"] for i in single.layer_info]
    # LPT balance: max load <= mean + largest unit (NS flops of the oracle's matrix list per group)
    cost = []
    for u in units:
        OL = _oracle_layer(cfg[u["layer"]])
        cost.append(sum(4.0 * max(M.m, M.n) * min(M.m, M.n) ** 2 for M in O.layer_matrices(OL)))
    loads = [sum(c for c, u in zip(cost, units) if u["owner"] == r) for r in range(world)]
    assert max(loads) <= sum(loads) / world + max(cost) * 1.5 + 1
    flops = [orth.orth_plan_query(p.h, "NS_FLOPS") for p in plans]
    assert abs(sum(flops) - orth.orth_plan_query(single.h, "NS_FLOPS")) <= world * 12


def test_host_only_plan_cannot_compute():
    p = orth.Plan(configs.cfg1(), device=-1)

    class Fake:
        def __init__(self, v): self.v = v
        def data_ptr(self): return self.v

    with pytest.raises(orth.OrthError) as ei:
        orth.orth_orthogonalize(p.h, Fake(256), Fake(512), stream=0)
    assert ei.value.status == orth.NO_DEVICE


def test_conv_scratch_sized_at_create():
    """SURVEY §8(b) "no call allocates after create": the per-layer conv scratch is derived from the
    declared grid and max_batch (host arithmetic, visible on a host-only plan), one slice per layer."""
    p0 = orth.Plan(configs.cfg2(), device=-1)
    assert all(i["scratch"] == 0 for i in p0.layer_info)                # max_batch 0: nothing declared
    p = orth.Plan(configs.cfg2(), device=-1, max_batch=256)
    sc = [i["scratch"] for i in p.layer_info]
    # 128 output channels at 16x16 (< 24 px): no padded copy; 512 @ 4x4 (2 x 2 x 16 tiles of 128 x 256 on
    # 148 SMs): split-K partials = tiles * 128 * 256 * 4 bytes
    tiles = (256 * 4 * 4 + 127) // 128 * (512 // 256)
    assert sc[10] == tiles * 128 * 256 * 4 and sc[11] == sc[10]
    p3 = orth.Plan(configs.cfg3(), device=-1, max_batch=256)
    s3 = [i["scratch"] for i in p3.layer_info]
    # cfg3 128-ch 28x28 layers take the stacked-window kernel, which loads its windows straight from the
    # input (no padded copy): no scratch
    assert s3[8] == 0
    # cfg3 512 @ 7x7: 98 x 2 = 196 tiles of 128 x 256 (1.32 waves on 148 SMs) split into K halves that fill
    # 2.65 waves: partials 196 x 128 x 256 x 4 bytes; at batch 32 (25 tiles <= 74) the few-tiles rule
    t3 = (256 * 7 * 7 + 127) // 128 * 2
    assert s3[28] == t3 * 128 * 256 * 4
    t32 = (32 * 7 * 7 + 127) // 128 * 2
    assert orth.Plan(configs.cfg3(), device=-1, max_batch=32).layer_info[28]["scratch"] == t32 * 128 * 256 * 4


def test_soc_validation_and_geometry():
    """f3: SOC layers need c_in == c_out, an odd kernel, stride 1 and 1 <= terms <= 16 (R27); the applied
    kernel is k_eff = terms (k - 1) + 1 with the centred padding, and the free kernel is one c/g x (c/g) k^2
    matrix per group (role K) that is not orthogonalised (no NS flops)."""
    for bad, st in [(dict(kind="soc", c_in=8, c_out=16, k=3), orth.UNSUPPORTED_CONFIG),
                    (dict(kind="soc", c_in=8, c_out=8, k=4), orth.UNSUPPORTED_CONFIG),
                    (dict(kind="soc", c_in=8, c_out=8, k=3, s=2), orth.UNSUPPORTED_CONFIG),
                    (dict(kind="soc", c_in=8, c_out=8, k=3, terms=40), orth.INVALID_ARGUMENT)]:
        assert orth.orth_validate_desc([dict(bad, padding_mode="circular")]) == st, bad
    p = orth.Plan([dict(kind="soc", c_in=32, c_out=32, k=3, s=1, d=2, g=2, terms=5, padding_mode="circular")], -1)
    assert p.layer_info[0]["k_eff"] == 11 and p.kernel_shape(0) == (32, 16, 11, 11)
    assert [(m["m"], m["n"], m["role"]) for m in p.matrices] == [(16, 144, "K"), (16, 144, "K")]
    assert p.ns_flops == 0 and p.out_hw(0, 12, 12) == (12, 12)
