"""Measurement of the SURVEY §8(f) rows on the GPU (one JSON line per row; CUDA events on the launching
stream, warm-up first, median of repeats).  Synthetic inputs shaped like the paper's workloads.

  f1 backward  : cfg3 (batch 256, BF16): weight gradient of every layer (tcgen05, TFLOP/s vs the BF16 burst
                 peak), the composition VJP and the orthogonalisation VJP of the whole network
  f2 certify   : cfg3 kernels on an 8 x 8 circular grid (FP64 Gram of the polyphase symbols; GFLOP/s)
  f3 SOC       : explicit exponential of 64/128/256-channel 3x3 kernels, 6 terms (construction GFLOP/s),
                 plus the apply of the 13 x 13 kernel vs the 6 implicit 3 x 3 convs it replaces
  f4 SLL block : fused block (C conv + concat + strided M conv) vs the three unfused convs, 128 -> 256 ch @ 32^2

Usage: python tools/bench_rows.py [--rows f1,f2,f3,f4] > profiles/r2_rows.jsonl
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs, gen  # noqa: E402
from tests.helpers import pack_params  # noqa: E402

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def construct(layers, compute="bf16", **kw):
    plan = orth.Plan(layers, 0, compute=compute, **kw)
    params, mats = pack_params(plan, 3)
    p = torch.from_numpy(params).cuda()
    ortho = torch.zeros_like(p)
    plan.orthogonalize(p, ortho)
    kf = torch.zeros(plan.kf32_numel, device="cuda")
    kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
    plan.compose(ortho, kf, kb)
    plan.check()
    return plan, p, ortho, kf, kb


def row_f1():
    layers = configs.cfg3()
    N = 256
    plan, p, ortho, kf, kb = construct(layers, vjp=1, max_batch=N)
    H = 224
    out = []
    total_fl, total_ms, dgrad_ms = 0.0, 0.0, 0.0
    per = []
    for l, d in enumerate(layers):
        Ho, _ = plan.out_hw(l, H, H)
        x = torch.randn(N, H, H, d["c_in"], device="cuda").to(torch.bfloat16)
        dy = torch.randn(N, Ho, Ho, d["c_out"], device="cuda").to(torch.bfloat16)
        dK = torch.zeros(plan.kernel_shape(l), device="cuda")
        nb = orth.orth_conv_wgrad_workspace(plan.h, l, N, H, H, orth.BF16)
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
        ms = timed(lambda: plan.conv_wgrad(l, x, dy, dK, workspace=ws))
        fl = 2.0 * N * Ho * Ho * d["c_out"] * d["c_in"] * d["k"] ** 2 / d["g"]
        kv = plan.kernel_bf16(kb, l)
        dx = torch.empty_like(x)
        ms_d = timed(lambda: plan.conv_transpose(l, kv, dy, dx))   # dgrad: the exact adjoint (a7)
        per.append(dict(layer=l, ms=ms, tflops=fl / ms / 1e9, dgrad_ms=ms_d, dgrad_tflops=fl / ms_d / 1e9))
        total_fl += fl
        total_ms += ms
        dgrad_ms += ms_d
        H = Ho
        del x, dy, dx
    dKall = torch.randn(plan.kf32_numel, device="cuda")
    dortho = torch.zeros_like(p)
    dparams = torch.zeros_like(p)
    ms_c = timed(lambda: plan.compose_vjp(ortho, dKall, dortho))
    ms_o = timed(lambda: plan.orthogonalize_vjp(p, dortho, dparams))
    plan.check()
    ach = total_fl / total_ms / 1e9
    out.append(dict(row="f1 backward", workload="config 3, batch 256, BF16", wgrad_ms_total=total_ms,
                    wgrad_tflops=ach, wgrad_frac_of_burst=ach / PEAKS["bf16_tflops"], wgrad_per_layer=per,
                    dgrad_ms_total=dgrad_ms, dgrad_tflops=total_fl / dgrad_ms / 1e9,
                    compose_vjp_ms=ms_c, orthogonalize_vjp_ms=ms_o,
                    note="VJP phases are the generic 3-pass tcgen05 GEMM (FP32-accurate), not the tuned forward kernels"))
    return out


def row_f2():
    layers = configs.cfg3()
    plan, p, ortho, kf, kb = construct(layers)
    res, tot_fl, tot_ms, worst = [], 0.0, 0.0, 0.0
    for l in [0, 1, 7, 8, 15, 16, 27, 28]:
        d = layers[l]
        K = plan.kernel_f32(kf, l).reshape(-1).contiguous()
        nb = orth.orth_certify_workspace(plan.h, l, 8, 8)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        outp = {}

        def run():
            outp["o"] = plan.certify(l, K, 8, 8, power_iters=30, workspace=ws)
        ms = timed(run, reps=5, warm=1)
        s = d["s"]
        ci_s, co = d["c_in"] * s * s, d["c_out"]
        S, Kd = min(co, ci_s), max(co, ci_s)
        F = (8 // s) ** 2
        fl = 8.0 * F * S * (S + 1) / 2 * Kd   # Hermitian complex FP64 Gram: 4 real FMAs per complex MAC
        tot_fl += fl
        tot_ms += ms
        worst = max(worst, float(outp["o"][..., 0].max()))
        res.append(dict(layer=l, ms=ms, gflops_fp64=fl / ms / 1e6, max_frob=float(outp["o"][..., 0].max())))
    return [dict(row="f2 certify", workload="config 3 kernels (BF16-mode construction), 8x8 circular grid",
                 per_layer=res, total_ms=tot_ms, gflops_fp64=tot_fl / tot_ms / 1e6, worst_certificate=worst,
                 note="FP64 SIMT (DFMA) Gram, upper-triangle tiles; bound: FP64 ALU, 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s")]


def row_f3():
    out = []
    for c in (64, 128, 256):
        layers = [dict(kind="soc", c_in=c, c_out=c, k=3, s=1, d=1, g=1, terms=6, padding_mode="circular", H=32)]
        plan, p, ortho, kf, kb = construct(layers, max_batch=256)
        ms = timed(lambda: plan.compose(ortho, kf, kb))
        fl = orth.orth_plan_query(plan.h, "COMP_FLOPS")
        x = torch.randn(256, 32, 32, c, device="cuda").to(torch.bfloat16)
        y = torch.empty_like(x)
        ms_apply = timed(lambda: plan.conv_forward(0, plan.kernel_bf16(kb, 0), x, y))
        # the implicit form ("needs to be done for each input"): 6 applications of a 3x3 conv
        p3 = orth.Plan([dict(kind="conv", c_in=c, c_out=c, k=3, s=1, d=1, g=1, padding_mode="circular", H=32)], 0,
                       max_batch=256)
        k3 = torch.randn(c, 3, 3, c, device="cuda").to(torch.bfloat16)
        ms_3 = timed(lambda: p3.conv_forward(0, k3, x, y))
        out.append(dict(row="f3 SOC", c=c, terms=6, k_eff=13, construct_ms=ms, construct_tflops=fl / ms / 1e9,
                        apply_13x13_ms=ms_apply, implicit_6x3x3_ms=6 * ms_3,
                        note="construction = batched block-conv GEMMs (3-pass tcgen05); the 13x13 apply runs on "
                             "the tcgen05 gather conv (k <= 13)"))
    return out


def row_f4():
    c, cs, co, H, N = 128, 128, 256, 32, 256
    layers = [dict(kind="conv", c_in=c, c_out=c, k=2, s=1, d=1, g=1, padding_mode="circular", H=H),
              dict(kind="sll", c_in=c, c_out=cs, k=2, s=1, d=1, g=1, padding_mode="circular", H=H),
              dict(kind="conv", c_in=c, c_out=co, k=3, s=2, d=1, g=1, padding_mode="circular", H=H),
              dict(kind="sll_block", c_in=c, c_out=co, k=1, s=2, d=1, g=1, padding_mode="circular", H=H,
                   pre=0, sll=1, post=2)]
    plan, p, ortho, kf, kb = construct(layers, max_batch=N)
    x = torch.randn(N, H, H, c, device="cuda").to(torch.bfloat16)
    y = torch.empty(N, H // 2, H // 2, co, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(cs, device="cuda")
    ms_f = timed(lambda: plan.conv_forward(3, plan.block_kernels(kb, 3)[0].reshape(-1), x, y, bias=b))
    t1 = torch.empty(N, H, H, c, device="cuda", dtype=torch.bfloat16)
    t2 = torch.empty(N, H, H, cs, device="cuda", dtype=torch.bfloat16)
    t3 = torch.empty(N, H, H, c, device="cuda", dtype=torch.bfloat16)

    def unfused():   # conv K_pre, conv K (+relu not fused), adjoint of K, conv K_post (stride 2)
        plan.conv_forward(0, plan.kernel_bf16(kb, 0), x, t1)
        plan.conv_forward(1, plan.kernel_bf16(kb, 1), t1, t2)
        plan.conv_transpose(1, plan.kernel_bf16(kb, 1), t2, t3)
        plan.conv_forward(2, plan.kernel_bf16(kb, 2), t3, y)
    ms_u = timed(unfused)
    ms_m = timed(lambda: plan.compose(ortho, kf, kb))
    plan.check()
    return [dict(row="f4 SLL x AOC block", workload=f"{c}->{co} ch, c_s {cs}, 2x2/2x2/3x3 s2 at {H}^2, batch {N}, BF16",
                 fused_forward_ms=ms_f, unfused_4_convs_ms=ms_u, construct_and_merge_ms=ms_m,
                 note="unfused = the three layers applied one after another (4 conv launches, no elementwise ops)")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="f1,f2,f3,f4")
    a = ap.parse_args()
    for r in a.rows.split(","):
        for line in {"f1": row_f1, "f2": row_f2, "f3": row_f3, "f4": row_f4}[r]():
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
