#!/usr/bin/env python
"""Benchmark of the orthogonal-conv hot path (BASELINE.json metric
"orth-conv layers/s (orthogonalize+compose+fwd), NS TFLOP/s vs peak, HBM GB/s").

One step = the whole hot path on one batch: orth_orthogonalize (power
pre-scaling + T Bjorck/NS iterations of every parameter matrix), orth_compose_kernel
(BCOP chain, RKO (*) BCOP, emit), then orth_conv_forward of every layer of the
network, chained, on the step's batch.  Workload (N=1): BASELINE configs[1] =
config 2 "CIFAR-AOC-12" (synth/configs.py), batch 256 at 32x32, bf16 NHWC
activations, FP32 construction.

value = layers/s = (#conv layers x ranks) / step time (weak scaling: every
rank runs the forward on its own batch of 256; construction is sharded by
layer across ranks and the BF16 kernels are NCCL-all-gathered).

Usage: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "orth-conv layers/s (orthogonalize+compose+fwd), NS TFLOP/s vs peak, HBM GB/s"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def start(self):
        """Start the 100 ms sampler; returns once it has produced its first line (nvidia-smi takes
        a few hundred ms to come up, longer than a short timed region)."""
        import threading
        self.lines, self.t0, self.t1 = [], None, None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
            return

        def reader():
            for line in self.p.stdout:
                self.lines.append((time.monotonic(), line))
        threading.Thread(target=reader, daemon=True).start()
        t_end = time.monotonic() + 5.0
        while not self.lines and time.monotonic() < t_end:
            time.sleep(0.01)

    def mark(self, begin: bool):
        """Bracket the sampled window (the timed region plus the load window after it)."""
        if begin:
            self.t0 = time.monotonic()
        else:
            self.t1 = time.monotonic()

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = (self.t1 if self.t1 is not None else time.monotonic()) + 0.1
        out = "".join(line for t, line in self.lines if t0 <= t <= t1)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "window": "timed region + the same step replayed untimed until >= 0.4 s (100 ms sampling)",
                "window_s": round(t1 - 0.1 - t0, 3) if self.t0 is not None else None}


def clock_window(clk, step, torch, min_s=0.4):
    """A timed region shorter than a few nvidia-smi periods (cfg2: 20 x 0.85 ms) gets no clock
    sample of its own, so the sampled window is the timed region plus the same step, untimed,
    repeated right after it until the window spans min_s seconds."""
    if clk.t0 is not None:
        while time.monotonic() - clk.t0 < min_s:
            for _ in range(8):
                step()
            torch.cuda.synchronize()
    clk.mark(False)


# ------------------------------------------------------------------ workload
def build_workload(orth, torch, cfg_layers, rank, world, device, compute, batch, chain=True, cfg_id=2,
                   plan_rank=None, plan_world=None):
    """Plan, seeded parameters / power vectors, activations.  chain: each
    layer consumes the previous output (cfg2/cfg3); otherwise every layer gets
    its own seeded input (cfg4).  A transposed layer's forward is
    orth_conv_transpose (small -> large grid)."""
    from synth import gen
    plan = orth.Plan(cfg_layers, device, rank=rank if plan_rank is None else plan_rank,
                     world=world if plan_world is None else plan_world, compute=compute, max_batch=max(batch, 0))
    params = np.zeros(plan.params_numel, np.float32)
    dev = torch.device("cuda", device)
    for i, m in enumerate(plan.matrices):
        key = (cfg_id, m["layer"], m["group"], i, gen.ROLE_ID[m["role"]])
        if m["m"] * m["n"] > (1 << 21):   # large dense sweep matrices: same recipe, QR on the GPU
            A = gen.param_matrix_torch(m["m"], m["n"], key, torch, dev).cpu().numpy()
        else:
            A = gen.param_matrix(m["m"], m["n"], key)
        params[m["off"]: m["off"] + A.size] = A.ravel()
    cache = np.zeros(plan.cache_numel, np.float32)
    for i, m in enumerate(plan.matrices):
        v = gen.unit_vector(m["n"], (cfg_id, m["layer"], m["group"], i, gen.ROLE_ID["v"]))
        cache[m["cache_off"]: m["cache_off"] + v.size] = v
    W = dict(plan=plan, params_h=params, cache_h=cache, chain=chain)
    W["params"] = torch.from_numpy(params).to(dev)
    W["cache"] = torch.from_numpy(cache).to(dev)
    W["ortho"] = torch.zeros_like(W["params"])
    W["kf32"] = torch.zeros(plan.kf32_numel, device=dev)
    W["kbf16"] = torch.zeros(plan.kbf16_numel, device=dev, dtype=torch.bfloat16)
    ins, acts, shapes = [], [], []
    H = cfg_layers[0]["H"]
    if batch == 0:       # dense NS sweep (config 5): construction only
        cfg_layers = []
        W["x_h"] = np.zeros((1,), np.float32)
    for l, d in enumerate(cfg_layers):
        if not chain or l == 0:
            H = d["H"]
            xl = gen.activations((batch, H, H, d["c_in"]), (cfg_id, rank, l, 0, gen.ROLE_ID["x"]))
            if l == 0:
                W["x_h"] = xl
            ins.append(torch.from_numpy(xl).to(dev, torch.bfloat16))
        else:
            ins.append(acts[-1])
        if d.get("kind") == "convT":
            Ho = H * d["s"]                       # large grid of the transposed layer
        else:
            Ho, _ = plan.out_hw(l, H, H)
        acts.append(torch.empty((batch, Ho, Ho, d["c_out"]), device=dev, dtype=torch.bfloat16))
        shapes.append((H, Ho, d))
        H = Ho
    W["x"] = ins[0] if ins else torch.zeros(1, device=dev, dtype=torch.bfloat16)
    W["ins"], W["acts"], W["shapes"] = ins, acts, shapes
    W["kviews"] = [plan.kernel_bf16(W["kbf16"], l) for l in range(len(cfg_layers))]
    return W


def conv_flops_bytes(shapes, batch):
    """Algorithmic flops / bytes of each layer apply (a6 / a7)."""
    fl, by = [], []
    for (H, Ho, d) in shapes:
        ci, co, k, g = d["c_in"], d["c_out"], d["k"], d["g"]
        small = H if d.get("kind") == "convT" else Ho       # output grid of the forward conv
        fl.append(2.0 * batch * small * small * co * (ci // g) * k * k)
        by.append(2.0 * batch * (H * H * ci + Ho * Ho * co) + 2.0 * co * (ci // g) * k * k)
    return fl, by


def apply_layer(W, l):
    plan = W["plan"]
    if W["shapes"][l][2].get("kind") == "convT":
        plan.conv_transpose(l, W["kviews"][l], W["ins"][l], W["acts"][l])
    else:
        plan.conv_forward(l, W["kviews"][l], W["ins"][l], W["acts"][l])


def run_step(W, orth, torch, world, pg, ev=None, graphs=None):
    """One step.  ev: optional dict of event lists to time the phases.
    graphs: optional CUDA graphs of the phases (captured from these same calls)."""
    plan = W["plan"]
    rec = (lambda name: ev[name].append(torch.cuda.Event(enable_timing=True)) or ev[name][-1].record()) \
        if ev is not None else (lambda name: None)
    rec("orth0")
    if graphs:
        graphs["orth"].replay()
    else:
        plan.orthogonalize(W["params"], W["ortho"], W["cache"])
    rec("orth1")
    if graphs:
        graphs["comp"].replay()
    else:
        plan.compose(W["ortho"], W["kf32"], W["kbf16"])
    rec("comp1")
    if world > 1 and W.get("sharded", True):
        from paper_2601_13776_b200.dist import gather_kernels
        gather_kernels(plan, W["kbf16"], orth.orth_plan_query(plan.h, "KERNEL_SEGMENT_BF16"), pg)
    rec("gather1")
    for l in range(len(W["acts"])):
        rec(f"conv{l}_0")
        if graphs:
            graphs[f"conv{l}"].replay()
        else:
            apply_layer(W, l)
        rec(f"conv{l}_1")
    return W["acts"][-1] if W["acts"] else W["ortho"]


def capture_graphs(W, torch):
    """One CUDA graph per phase (orthogonalize, compose, one per layer apply),
    captured from the library's own calls on the capture stream."""
    plan = W["plan"]
    graphs = {}
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            plan.orthogonalize(W["params"], W["ortho"], W["cache"])
        graphs["orth"] = g
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            plan.compose(W["ortho"], W["kf32"], W["kbf16"])
        graphs["comp"] = g
        for l in range(len(W["acts"])):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                apply_layer(W, l)
            graphs[f"conv{l}"] = g
        # the whole step as ONE graph (what a serving loop replays): the timed steps use it;
        # the per-phase graphs above only serve the breakdown
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            plan.orthogonalize(W["params"], W["ortho"], W["cache"])
            plan.compose(W["ortho"], W["kf32"], W["kbf16"])
            for l in range(len(W["acts"])):
                apply_layer(W, l)
        graphs["step"] = g
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return graphs


def ours(args):
    import torch
    import paper_2601_13776_b200 as orth
    from synth import configs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD
    if args.config == 5:
        cfg, batch = configs.cfg5(args.n)[: args.mats], 0
    else:
        cfg = configs.CONFIGS[args.config]()
        batch = configs.BATCH[args.config]
    # construction: sharded by layer + all-gather, or replicated on every rank (no collective; SURVEY 8(e):
    # cfg2/cfg3 construction is latency-bound, so sharding saves little there)
    mode = args.construct if args.construct != "auto" else ("sharded" if args.config == 5 else "replicated")
    sharded = world > 1 and mode == "sharded"
    W = build_workload(orth, torch, cfg, rank, world, local, args.compute, batch,
                       chain=configs.CHAIN.get(args.config, False), cfg_id=args.config,
                       plan_rank=rank if sharded else 0, plan_world=world if sharded else 1)
    W["sharded"] = sharded
    plan = W["plan"]
    flush = torch.empty(int(2 * 126e6 // 4) + 1024, device="cuda", dtype=torch.float32)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        l0 = plan.launches
        run_step(W, orth, torch, world, pg)
        per_step_launches = plan.launches - l0
    plan.check()
    barrier()
    graphs = capture_graphs(W, torch) if (not sharded and not args.no_graph) else None
    if graphs:
        for _ in range(2):
            run_step(W, orth, torch, world, pg, graphs=graphs)
        barrier()
    clk = Clocks(local)
    clk.start()
    launches0 = plan.launches
    nl = len(W["acts"])
    names = ["orth0", "orth1", "comp1", "gather1"] + [f"conv{l}_{e}" for l in range(nl) for e in (0, 1)]
    ev = {n: [] for n in names}
    barrier()
    clk.mark(True)
    if graphs:
        # timed region: K steps, each one graph replay bracketed by events (L2 flushed before each)
        s_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()                              # L2 flush outside the events
            s_ev[i][0].record()
            graphs["step"].replay()
            s_ev[i][1].record()
        barrier()
        clock_window(clk, lambda: (flush.zero_(), graphs["step"].replay()), torch)
        clocks = clk.stop()
        step_ms = [a.elapsed_time(b) for a, b in s_ev]
        # breakdown (untimed for `value`): the same K steps through the per-phase graphs
        for _ in range(args.steps):
            flush.zero_()
            run_step(W, orth, torch, world, pg, ev, graphs)
        barrier()
    else:
        for _ in range(args.steps):
            flush.zero_()                              # L2 flush outside the events
            run_step(W, orth, torch, world, pg, ev, graphs)
        barrier()
        clock_window(clk, lambda: (flush.zero_(), run_step(W, orth, torch, world, pg, None, graphs)), torch)
        clocks = clk.stop()
    launches = plan.launches - launches0 if not graphs else per_step_launches * args.steps
    plan.check()
    el = lambda a, b, i: ev[a][i].elapsed_time(ev[b][i])
    last = f"conv{nl - 1}_1" if nl else "gather1"
    if not graphs:
        step_ms = [el("orth0", last, i) for i in range(args.steps)]
    t_step = sum(step_ms) / args.steps
    t_orth = sum(el("orth0", "orth1", i) for i in range(args.steps)) / args.steps
    t_comp = sum(el("orth1", "comp1", i) for i in range(args.steps)) / args.steps
    t_gather = sum(el("comp1", "gather1", i) for i in range(args.steps)) / args.steps
    t_conv = [sum(el(f"conv{l}_0", f"conv{l}_1", i) for i in range(args.steps)) / args.steps for l in range(nl)]
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([t_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())
    fl, by = conv_flops_bytes(W["shapes"], batch)
    P = peaks()
    ns_flops = orth.orth_plan_query(plan.h, "NS_FLOPS")
    # dominant kernel class: conv forward (sum over layers) vs NS.  `traffic`: DRAM bytes per launch of
    # that class from the committed ncu --set full capture of the same workload (profiles/r1_traffic.json)
    traffic_db = {}
    try:
        traffic_db = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                                 "r1_traffic.json")))
    except (OSError, ValueError):
        pass
    wl = traffic_db.get(configs.NAMES.get(args.config, ""), {})

    def traffic(kind):
        t = wl.get(kind)
        return t["dram_bytes_per_launch"] if t else None
    conv_total = sum(t_conv)
    if nl and conv_total >= t_orth:
        ach = sum(fl) / (conv_total * 1e-3) / 1e12
        roof = {"kernel": f"conv apply (orth_conv_forward / orth_conv_transpose), {len(fl)} launches", "bound": "tensor", "achieved": ach,
                "peak": P["bf16_tflops_sustained"], "unit": "TFLOP/s", "frac": ach / P["bf16_tflops_sustained"],
                "traffic": traffic("conv apply"), "traffic_source": wl.get("source"),
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                "per_launch_flops_avg": sum(fl) / len(fl), "avg_launch_ms": conv_total / len(fl),
                "share_of_step": conv_total / t_step}
    else:
        ach = ns_flops / (t_orth * 1e-3) / 1e12
        roof = {"kernel": "orth_orthogonalize (power + NS)", "bound": "tensor", "achieved": ach,
                "peak": P["bf16_tflops_sustained"], "unit": "TFLOP/s", "frac": ach / P["bf16_tflops_sustained"],
                "traffic": traffic("orth_orthogonalize (power + NS)"), "traffic_source": wl.get("source"),
                "share_of_step": t_orth / t_step}
    # ---- e2e through the public API with host buffers
    e2e = e2e_run(W, orth, torch, world, pg, args, barrier)
    out = {
        "metric": METRIC, "value": len(cfg) * world / (t_step * 1e-3), "unit": "layers/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": {"bf16": "bf16", "bf16x3": "bf16x3", "f32": "f32+bf16"}[args.compute],
        "data": "synthetic (seeded near-orthogonal params, N(0,1) activations; SURVEY §8(d))",
        "config": {"workload": configs.NAMES.get(args.config, f"config 5: {len(cfg)} dense {args.n}x{args.n} matrices"),
                   "global_batch": batch * world, "per_rank_batch": batch, "image": cfg[0]["H"], "ns_iters": 12,
                   "construction": {"f32": "FP32 FFMA (SIMT)",
                                    "bf16": "tcgen05 BF16, FP32 master, 3-pass split polish + composition",
                                    "bf16x3": "tcgen05 3-pass hi/lo split everywhere"}[args.compute],
                   "activations": "bf16 NHWC",
                   "parallelism": f"dp{world} (construction " + ("sharded by layer + all-gather)" if sharded else
                                                                 "replicated on every rank, no collective)"),
                   "l2": "flushed between timed steps (252 MB write)",
                   "launch": ("one CUDA graph per step (per-phase graphs for the breakdown)" if graphs
                              else "eager")},
        "breakdown_ms": {"orthogonalize": t_orth, "compose": t_comp, "allgather": t_gather,
                         "conv_forward": conv_total, "conv_per_layer": t_conv},
        "construction_layers_per_s": len(cfg) / ((t_orth + t_comp + t_gather) * 1e-3),
        "ns_tflops": ns_flops / (t_orth * 1e-3) / 1e12,
        "conv_tflops": sum(fl) / (conv_total * 1e-3) / 1e12 if nl else None,
        "conv_gbs": sum(by) / (conv_total * 1e-3) / 1e9 if nl else None,
        "roofline": roof,
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in (1, 2):
        out["cpu_baseline"] = cpu_baseline(args, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def e2e_run(W, orth, torch, world, pg, args, barrier):
    """Same step through the public API with HOST buffers: pinned H2D of every
    step's inputs (params + x) and D2H of its result inside the timed region.
    Graph mode runs the loop a serving process would: two input / result buffer
    sets, the copies on their own stream, so step i+1's H2D and step i's D2H
    overlap step i's compute (each step still copies its own inputs and result)."""
    ph = torch.from_numpy(W["params_h"]).pin_memory()
    xh = torch.from_numpy(W["x_h"]).to(torch.bfloat16).pin_memory()
    res = W["acts"][-1] if W["acts"] else W["ortho"]
    s = torch.cuda.current_stream()
    n = max(1, args.steps)
    out = {"h2d_bytes_per_step": int(ph.numel() * 4 + xh.numel() * 2)}
    if args.no_graph or W.get("sharded", False):
        yh = torch.empty(res.shape, dtype=res.dtype).pin_memory()

        def step():
            W["params"].copy_(ph, non_blocking=True)   # H2D of this step's parameters and input batch
            W["x"].copy_(xh, non_blocking=True)
            run_step(W, orth, torch, world, pg)
            yh.copy_(res, non_blocking=True)           # D2H of the result
        for _ in range(2):
            step()
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s)
        for _ in range(n):
            step()
        t1.record(s)
        barrier()
        ms = t0.elapsed_time(t1) / n
        out.update(launch="eager, serial copies", d2h_bytes_per_step=int(yh.numel() * yh.element_size()))
    else:
        plan = W["plan"]
        P = [W["params"], torch.empty_like(W["params"])]
        X = [W["x"], torch.empty_like(W["x"])]
        Y = [torch.empty_like(res), torch.empty_like(res)]              # device copies of each step's result
        yh = [torch.empty(res.shape, dtype=res.dtype).pin_memory() for _ in range(2)]
        x0 = W["ins"][0] if W["ins"] else None
        torch.cuda.synchronize()
        cs = torch.cuda.Stream()
        graphs = []
        for b in range(2):   # one compute graph per buffer set
            W["params"] = P[b]
            if W["ins"]:
                W["ins"][0] = X[b]
            cs.wait_stream(s)
            with torch.cuda.stream(cs):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    run_step(W, orth, torch, world, pg)
                    Y[b].copy_(res)
            s.wait_stream(cs)
            graphs.append(g)
        W["params"] = P[0]
        if W["ins"]:
            W["ins"][0] = x0
        torch.cuda.synchronize()
        c = torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def loop(steps):
            c.wait_stream(s)
            with torch.cuda.stream(c):                # inputs of step 0
                P[0].copy_(ph, non_blocking=True)
                X[0].copy_(xh, non_blocking=True)
                ev_in[0].record(c)
            for i in range(steps):
                b = i % 2
                if i + 1 < steps:                     # prefetch step i+1's inputs into the other set
                    with torch.cuda.stream(c):
                        if i >= 1:
                            c.wait_event(ev_done[1 - b])   # step i-1 has finished reading that set
                        P[1 - b].copy_(ph, non_blocking=True)
                        X[1 - b].copy_(xh, non_blocking=True)
                        ev_in[1 - b].record(c)
                s.wait_event(ev_in[b])
                if i >= 2:
                    s.wait_event(ev_out[b])           # Y[b] of step i-2 has reached the host
                graphs[b].replay()
                ev_done[b].record(s)
                with torch.cuda.stream(c):            # D2H of step i's result
                    c.wait_event(ev_done[b])
                    yh[b].copy_(Y[b], non_blocking=True)
                    ev_out[b].record(c)
            s.wait_stream(c)
        loop(2)
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s)
        loop(n)
        t1.record(s)
        barrier()
        ms = t0.elapsed_time(t1) / n
        out.update(launch="CUDA graph per step; H2D of step i+1 and D2H of step i on a copy stream, overlapping "
                          "step i's compute (two buffer sets)",
                   d2h_bytes_per_step=int(Y[0].numel() * Y[0].element_size()))
        W["e2e_result"] = yh[(n - 1) % 2]
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out.update(value=len(W["plan"].layers) * world / (ms * 1e-3), unit="layers/s", ms_per_step=ms)
    return out


# ------------------------------------------------------------------ oracle (CPU) legs
def _oracle_step(cfg, batch, n_img, seed_cfg=2):
    """Oracle step on a bounded sample: full construction (all matrices) and the
    forward of n_img images, extrapolated to the batch.  Returns (t_equiv_s, t_construct_s, t_img_s)."""
    import oracle as O
    from synth import gen
    from tests.helpers import oracle_construct, oracle_layer
    mats = []
    i = 0
    for l, d in enumerate(cfg):
        OL = oracle_layer(d)
        for g in range(OL.g):
            for M in O.layer_matrices(OL):
                mats.append(gen.param_matrix(M.m, M.n, (seed_cfg, l, g, i, gen.ROLE_ID[M.role])))
                i += 1
    t0 = time.perf_counter()
    _, _, ks = oracle_construct(cfg, mats)
    t1 = time.perf_counter()
    x = gen.activations((n_img, cfg[0]["c_in"], cfg[0]["H"], cfg[0]["H"]), (seed_cfg, 0, 0, 0, 6)).astype(np.float64)
    for l, d in enumerate(cfg):
        OL = oracle_layer(d)
        x = O.conv2d(x, ks[l], s=OL.s, d=OL.d, g=OL.g)
    t2 = time.perf_counter()
    t_img = (t2 - t1) / n_img
    return (t1 - t0) + batch * t_img, t1 - t0, t_img


def _threads():
    n = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(n)
    except Exception:
        pass
    return n


def cpu_baseline(args, budget_s=30.0):
    from synth import configs
    cores = _threads()
    cfg = configs.CONFIGS[args.config]()
    batch = configs.BATCH[args.config]
    t_eq, t_c, t_img = _oracle_step(cfg, batch, 1)
    return {"value": len(cfg) / t_eq, "unit": "layers/s", "cores": cores, "kind": "oracle",
            "sample": f"config {args.config}: full oracle construction ({t_c:.2f} s, all matrices, T=12, float64) + "
                      f"forward of 1 image ({t_img:.2f} s) extrapolated to batch {batch}",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def reference(args):
    """The oracle as the reference arm (tier framing: the CPU float64 oracle)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import configs
    cores = _threads()
    cfg = configs.CONFIGS[args.config]()
    batch = configs.BATCH[args.config]
    for _ in range(min(args.warmup, 1)):
        _oracle_step(cfg, batch, 1)
    ts = []
    for _ in range(args.steps):
        t_eq, t_c, t_img = _oracle_step(cfg, batch, 1)
        ts.append(t_eq)
    t = sum(ts) / len(ts)
    v = len(cfg) / t
    out = {"metric": METRIC, "value": v, "unit": "layers/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": configs.NAMES[args.config], "global_batch": batch},
           "cpu_baseline": {"value": v, "unit": "layers/s", "cores": cores, "kind": "oracle",
                            "sample": f"each step: full float64 oracle construction + forward of 1 image "
                                      f"extrapolated to batch {batch}", "cpu": _cpu_model()},
           "e2e": {"value": v, "unit": "layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=2048, help="config 5: matrix size")
    ap.add_argument("--mats", type=int, default=64, help="config 5: number of n x n matrices")
    ap.add_argument("--compute", default="bf16", choices=["f32", "bf16", "bf16x3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying CUDA graphs")
    ap.add_argument("--cpu-budget", type=float, default=30.0)
    ap.add_argument("--construct", default="auto", choices=["auto", "sharded", "replicated"],
                    help="N > 1: shard construction by layer + all-gather, or replicate it (auto: cfg5 sharded)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
