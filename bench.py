#!/usr/bin/env python
"""Benchmark of the orthogonal-conv hot path (BASELINE.json metric
"orth-conv layers/s (orthogonalize+compose+fwd), NS TFLOP/s vs peak, HBM GB/s").

One step = the whole hot path on one batch: orth_orthogonalize (power
pre-scaling + T Bjorck/NS iterations of every parameter matrix),
orth_compose_kernel (BCOP chain, RKO (*) BCOP, emit), for N > 1 the NCCL
all-gather of the kernel segments + orth_kernels_assemble, then
orth_conv_forward of every layer of the network, chained, on the step's batch.

Workload (N = 1, default): BASELINE configs[2] = config 3, the ImageNet
AOC-ResNet34-shape network (33 orthogonal convs, 224x224, batch 256) -- the
north star's target and the largest single-GPU configuration.  BF16
activations, BF16 tensor-core construction (FP32 master, split-precision
polish).  --config 2 / 4 / 5 select the other BASELINE configurations.

N > 1 (--gpus N; relaunches itself under torch.distributed.run when WORLD_SIZE
is unset): STRONG scaling of the same job -- global batch 256 split over the
ranks, construction sharded by (layer, group) unit (LPT) with one in-place
all-gather of the BF16 kernel segments per step; value = layers / step time,
max over ranks.

Usage: python bench.py [--gpus N --steps K --warmup W] [--config C] [--impl reference]
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
GLOBAL_BATCH = 256


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        d["_source"] = "MEASURED_PEAKS.json"
        return d
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "_source": "fallback of /opt/skills/guides/B200_PROFILING.md"}


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.t0 = self.t1 = None

    def start(self):
        """Start the 100 ms sampler; returns once it has produced its first line."""
        import threading
        self.lines = []
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
    """A timed region shorter than a few nvidia-smi periods gets no clock sample of its own, so the
    sampled window is the timed region plus the same step, untimed, repeated until it spans min_s."""
    if clk.t0 is not None:
        while time.monotonic() - clk.t0 < min_s:
            for _ in range(4):
                step()
            torch.cuda.synchronize()
    clk.mark(False)


# ------------------------------------------------------------------ workload
class Workload:
    """Plan, seeded parameters / power vectors, activations of one rank."""

    def __init__(self, orth, torch, cfg_id, n, mats, rank, world, sharded, compute, device):
        from synth import configs, gen
        self.torch, self.orth = torch, orth
        self.cfg_id, self.rank, self.world = cfg_id, rank, world
        self.sharded = sharded and world > 1
        if cfg_id == 5:
            self.layers, self.batch, self.chain = configs.cfg5(n)[:mats], 0, False
            self.name = f"config 5: {len(self.layers)} dense {n}x{n} matrices (OrthoLinear), construction only"
        else:
            self.layers = configs.CONFIGS[cfg_id]()
            per = (GLOBAL_BATCH + world - 1) // world          # strong scaling: the global batch is split
            self.batch = min(per, GLOBAL_BATCH - rank * per)
            self.chain = configs.CHAIN[cfg_id]
            self.name = configs.NAMES[cfg_id]
        p_rank, p_world = (rank, world) if self.sharded else (0, 1)
        self.plan = plan = orth.Plan(self.layers, device, rank=p_rank, world=p_world, compute=compute,
                                     max_batch=max(self.batch, 0))
        dev = torch.device("cuda", device)
        params = np.zeros(plan.params_numel, np.float32)
        for i, m in enumerate(plan.matrices):
            key = (cfg_id, m["layer"], m["group"], i, gen.ROLE_ID[m["role"]])
            if m["m"] * m["n"] > (1 << 21):   # large dense-sweep matrices: same recipe, QR on the GPU
                A = gen.param_matrix_torch(m["m"], m["n"], key, torch, dev).cpu().numpy()
            else:
                A = gen.param_matrix(m["m"], m["n"], key)
            params[m["off"]: m["off"] + A.size] = A.ravel()
        cache = np.zeros(plan.cache_numel, np.float32)
        for i, m in enumerate(plan.matrices):
            v = gen.unit_vector(m["n"], (cfg_id, m["layer"], m["group"], i, gen.ROLE_ID["v"]))
            cache[m["cache_off"]: m["cache_off"] + v.size] = v
        self.params_h = params
        self.params = torch.from_numpy(params).to(dev)
        self.cache = torch.from_numpy(cache).to(dev)
        self.ortho = torch.zeros_like(self.params)
        self.kf32 = torch.zeros(plan.kf32_numel, device=dev)
        self.kbf16 = torch.zeros(plan.kbf16_numel, device=dev, dtype=torch.bfloat16)
        if self.sharded:   # gather layout: this rank's units in its segment, all-gathered every step
            self.gf32 = torch.zeros(plan.gf32_numel, device=dev)
            self.gbf16 = torch.zeros(plan.gbf16_numel, device=dev, dtype=torch.bfloat16)
        self.ins, self.acts, self.shapes = [], [], []
        H = self.layers[0]["H"] if self.layers else 0
        for l, d in enumerate(self.layers if self.batch > 0 else []):
            if not self.chain or l == 0:
                H = d["H"]
                xl = gen.activations((self.batch, H, H, d["c_in"]), (cfg_id, rank, l, 0, gen.ROLE_ID["x"]))
                if l == 0:
                    self.x_h = xl
                self.ins.append(torch.from_numpy(xl).to(dev, torch.bfloat16))
            else:
                self.ins.append(self.acts[-1])
            Ho = H * d["s"] if d.get("kind") == "convT" else plan.out_hw(l, H, H)[0]
            self.acts.append(torch.empty((self.batch, Ho, Ho, d["c_out"]), device=dev, dtype=torch.bfloat16))
            self.shapes.append((H, Ho, d))
            H = Ho
        if not self.ins:
            self.x_h = np.zeros((1,), np.float32)
        self.kviews = [plan.kernel_bf16(self.kbf16, l) for l in range(len(self.shapes))]

    # the three parts of a step (each graph-capturable; the all-gather between them is NCCL)
    def construct(self):
        p = self.plan
        p.orthogonalize(self.params, self.ortho, self.cache)
        if self.sharded:
            p.compose(self.ortho, self.gf32, self.gbf16)
        else:
            p.compose(self.ortho, self.kf32, self.kbf16)

    def gather(self, pg):
        from paper_2601_13776_b200.dist import gather_kernels
        gather_kernels(self.gbf16, self.plan.seg_bf16, pg)

    def apply(self, l):
        p = self.plan
        if self.shapes[l][2].get("kind") == "convT":
            p.conv_transpose(l, self.kviews[l], self.ins[l], self.acts[l])
        else:
            p.conv_forward(l, self.kviews[l], self.ins[l], self.acts[l])

    def forward(self):
        if self.sharded:   # a8: gathered segments -> contiguous per-layer BF16 kernels
            self.plan.assemble(None, None, self.gbf16, self.kbf16)
        for l in range(len(self.shapes)):
            self.apply(l)

    def result(self):
        return self.acts[-1] if self.acts else self.ortho


def capture(torch, fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return g


def conv_flops_bytes(shapes, batch):
    """Algorithmic flops / bytes of each layer apply (a6 / a7)."""
    fl, by = [], []
    for (H, Ho, d) in shapes:
        ci, co, k, g = d["c_in"], d["c_out"], d["k"], d["g"]
        small = H if d.get("kind") == "convT" else Ho       # output grid of the forward conv
        fl.append(2.0 * batch * small * small * co * (ci // g) * k * k)
        by.append(2.0 * batch * (H * H * ci + Ho * Ho * co) + 2.0 * co * (ci // g) * k * k)
    return fl, by


def trace_pass(W, steps):
    """Eager profiling pass (outside the timed region): the library's own trace (CUDA events around every
    kernel group it launches) over `steps` steps; returns the per-step lists of records."""
    plan = W.plan
    plan.trace(True)
    recs = []
    for _ in range(steps):
        W.construct()
        W.forward()
        recs.append(plan.trace_read())
    plan.trace(False)
    return recs


def roofline_blocks(W, orth, recs, P, traffic_db):
    """Dominant single kernel (largest share of the traced step) against the BURST bf16 peak (each traced
    group is timed alone), and the HBM-bound groups against the measured copy bandwidth."""
    plan = W.plan
    n = len(recs)
    fl, by = conv_flops_bytes(W.shapes, W.batch)
    groups = {}
    for step in recs:
        for r in step:
            key = r["variant"] if r["kind"] in ("conv_fwd", "conv_adj") else r["kind"]
            g = groups.setdefault(key, dict(ms=0.0, calls=0, launches=0, flops=0.0, bytes=0.0, layers=set()))
            g["ms"] += r["ms"] / n
            g["calls"] += 1.0 / n
            g["launches"] += r["launches"] / n
            if r["layer"] >= 0:
                g["flops"] += fl[r["layer"]] / n
                g["bytes"] += by[r["layer"]] / n
                g["layers"].add(r["layer"])
    if "ns" in groups:
        groups["ns"]["flops"] = orth.orth_plan_query(plan.h, "NS_FLOPS")
    if "compose" in groups:
        groups["compose"]["flops"] = orth.orth_plan_query(plan.h, "COMP_FLOPS")
    # algorithmic bytes of the bandwidth-bound groups: power mn*4*P (one read of W per
    # iteration), scale mn*(4 read + 4 write + 2 + 2 BF16 hi/lo), emit co*ci*k^2*(4 read + 4 + 2 written)
    mn = sum(m["m"] * m["n"] for m in plan.matrices)
    if "power" in groups:
        groups["power"]["bytes"] = mn * 4.0 * 3
    if "scale" in groups:
        groups["scale"]["bytes"] = mn * 12.0
    if "emit" in groups:
        groups["emit"]["bytes"] = sum(u["numel"] for u in plan.units) * 10.0
    total = sum(g["ms"] for g in groups.values())
    dom_key = max(groups, key=lambda k: groups[k]["ms"])
    d = groups[dom_key]
    hbm_like = {"power", "scale", "emit", "assemble", "ns_check", orth.CONV_VARIANTS[2], orth.CONV_VARIANTS[3]}

    def tr(name):
        t = traffic_db.get(name)
        return t.get("dram_bytes_per_launch") if isinstance(t, dict) else None
    if dom_key not in hbm_like and d["flops"] > 0:
        ach = d["flops"] / (d["ms"] * 1e-3) / 1e12
        roof = {"kernel": dom_key, "bound": "tensor", "achieved": ach, "peak": P["bf16_tflops"],
                "unit": "TFLOP/s", "frac": ach / P["bf16_tflops"], "traffic": tr(dom_key),
                "peak_source": f"{P['_source']} bf16_tflops (burst: each traced call is timed alone)",
                "frac_vs_sustained": ach / P["bf16_tflops_sustained"],
                "algorithmic_flops_per_launch": d["flops"] / max(d["calls"], 1e-9),
                "avg_launch_ms": d["ms"] / max(d["calls"], 1e-9), "launches_per_step": d["calls"],
                "layers": sorted(d["layers"]), "share_of_traced_step": d["ms"] / total,
                "timing": "library trace (CUDA events on the launching stream around each call), eager pass "
                          "after the timed region"}
    else:
        ach = d["bytes"] / (d["ms"] * 1e-3) / 1e9
        roof = {"kernel": dom_key, "bound": "hbm", "achieved": ach, "peak": P["hbm_gbs"], "unit": "GB/s",
                "frac": ach / P["hbm_gbs"], "traffic": tr(dom_key), "share_of_traced_step": d["ms"] / total}
    hbm = []
    for key in ["power", "scale", "emit", orth.CONV_VARIANTS[3], orth.CONV_VARIANTS[2]]:
        g = groups.get(key)
        if not g or g["bytes"] <= 0 or g["ms"] <= 0:
            continue
        gbs = g["bytes"] / (g["ms"] * 1e-3) / 1e9
        hbm.append({"kernel": key, "algorithmic_bytes_per_step": g["bytes"], "ms": g["ms"], "achieved": gbs,
                    "peak": P["hbm_gbs"], "unit": "GB/s", "frac": gbs / P["hbm_gbs"], "traffic": tr(key)})
    # grouped conv layers of cfg4 (g = 32: AI 144, HBM-bound by SURVEY §8(d))
    for l, (H, Ho, dsc) in enumerate(W.shapes):
        if dsc.get("g", 1) >= 32:
            ms = sum(r["ms"] for step in recs for r in step if r["layer"] == l) / n
            if ms > 0:
                gbs = by[l] / (ms * 1e-3) / 1e9
                hbm.append({"kernel": f"layer {l} grouped conv g={dsc['g']} "
                                      f"({'adjoint' if dsc.get('kind') == 'convT' else 'forward'})",
                            "algorithmic_bytes_per_step": by[l], "ms": ms, "achieved": gbs, "peak": P["hbm_gbs"],
                            "unit": "GB/s", "frac": gbs / P["hbm_gbs"], "tensor_tflops": fl[l] / (ms * 1e-3) / 1e12})
    table = {k: {"ms_per_step": v["ms"], "calls": v["calls"], "launches": v["launches"],
                 "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["flops"] and v["ms"] else None}
             for k, v in sorted(groups.items(), key=lambda kv: -kv[1]["ms"])}
    return roof, hbm, table


def ours(args):
    import torch
    import paper_2601_13776_b200 as orth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD
    sharded = world > 1 and args.construct != "replicated"
    W = Workload(orth, torch, args.config, args.n, args.mats, rank, world, sharded, args.compute, local)
    plan = W.plan
    flush = torch.empty(int(2 * 126e6 // 4) + 1024, device="cuda", dtype=torch.float32)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def eager_step():
        W.construct()
        if W.sharded:
            W.gather(pg)
        W.forward()

    per_step_launches = 0
    for _ in range(args.warmup):
        l0 = plan.launches
        eager_step()
        per_step_launches = plan.launches - l0
    plan.check()
    barrier()
    # CUDA graphs: the whole step as one graph (N = 1 or replicated construction); with the NCCL
    # all-gather, two graphs (construction | assemble + forward) around the eager collective
    if not args.no_graph:
        if W.sharded:
            gA, gB = capture(torch, W.construct), capture(torch, W.forward)

            def step():
                gA.replay()
                W.gather(pg)
                gB.replay()
            launch = "two CUDA graphs per step (construction | assemble + forward) around the NCCL all-gather"
        else:
            g_step = capture(torch, eager_step)
            step = g_step.replay
            launch = "one CUDA graph per step"
    else:
        step, launch = eager_step, "eager"
    for _ in range(2):
        step()
    barrier()
    clk = Clocks(local)
    clk.start()
    s_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    clk.mark(True)
    for i in range(args.steps):
        flush.zero_()                              # L2 flush outside the events
        s_ev[i][0].record()
        step()
        s_ev[i][1].record()
    barrier()
    clock_window(clk, lambda: (flush.zero_(), step()), torch)
    clocks = clk.stop()
    plan.check()
    t_step = sum(a.elapsed_time(b) for a, b in s_ev) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([t_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())
    P = peaks()
    # ---- breakdown: per-phase graphs (N = 1) timed with events, L2 flushed before each step
    breakdown = None
    if world == 1 and not args.no_graph:
        gc = capture(torch, W.construct)
        gl = [capture(torch, (lambda l=l: W.apply(l))) for l in range(len(W.shapes))]
        eo = []
        for _ in range(args.steps):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(gl) + 2)]
            ev[0].record()
            gc.replay()
            ev[1].record()
            for l, gg in enumerate(gl):
                gg.replay()
                ev[l + 2].record()
            eo.append(ev)
        torch.cuda.synchronize()
        t_cons = sum(e[0].elapsed_time(e[1]) for e in eo) / len(eo)
        t_conv = [sum(e[l + 1].elapsed_time(e[l + 2]) for e in eo) / len(eo) for l in range(len(gl))]
        breakdown = {"construction_ms": t_cons, "conv_forward_ms": sum(t_conv), "conv_per_layer_ms": t_conv,
                     "how": "per-phase CUDA graphs, CUDA events, L2 flushed before each step"}
    # ---- trace pass (eager, library events around each kernel group): dominant kernel + HBM-bound groups
    traffic_db = {}
    try:
        traffic_db = json.load(open(os.path.join(ROOT, "profiles", "r2_traffic.json"))).get(f"config {args.config}", {})
    except (OSError, ValueError):
        pass
    roof, hbm, table = None, [], None
    if world == 1:
        recs = trace_pass(W, max(3, min(args.steps, 10)))
        roof, hbm, table = roofline_blocks(W, orth, recs, P, traffic_db)
    ns_fl = orth.orth_plan_query(plan.h, "NS_FLOPS")
    ns_ms = table.get("ns", {}).get("ms_per_step") if table else None
    # ---- e2e through the public API with host buffers
    e2e = e2e_run(W, torch, world, pg, args, barrier, not args.no_graph)
    n_layers = len(W.layers)
    out = {
        "metric": METRIC, "value": n_layers / (t_step * 1e-3), "unit": "layers/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": {"bf16": "bf16", "bf16x3": "bf16x3", "f32": "f32+bf16"}[args.compute],
        "data": "synthetic (seeded near-orthogonal params, N(0,1) activations; SURVEY §8(d)); no trained weights",
        "config": {"workload": W.name, "global_batch": GLOBAL_BATCH if W.batch else 0, "per_rank_batch": W.batch,
                   "image": W.layers[0].get("H") if W.batch else None, "ns_iters": 12,
                   "construction": {"f32": "FP32 FFMA (SIMT)",
                                    "bf16": "tcgen05 BF16, FP32 master, 3-pass split polish + composition",
                                    "bf16x3": "tcgen05 3-pass hi/lo split everywhere"}[args.compute],
                   "activations": "bf16 NHWC",
                   "parallelism": (f"dp{world}: batch split over ranks; construction sharded by (layer, group) unit "
                                   "(LPT) + in-place NCCL all-gather of the BF16 kernel segments + assemble"
                                   if W.sharded else (f"dp{world}: batch split; construction replicated" if world > 1
                                                      else "1 GPU")),
                   "l2": "flushed between timed steps (252 MB write, outside the events)",
                   "launch": launch},
        "breakdown": breakdown,
        "kernel_groups_ms": table,
        "ns_tflops": (ns_fl / (ns_ms * 1e-3) / 1e12) if ns_ms else None,
        "roofline": roof,
        "roofline_hbm": hbm,
        "gpu_launches": per_step_launches * args.steps,
        "clocks": clocks,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in (1, 2, 3, 4):
        out["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def e2e_run(W, torch, world, pg, args, barrier, graphs_ok):
    """Same step through the public API with HOST buffers: pinned H2D of every step's inputs (params + x)
    and D2H of its result inside the timed region.  Run as a serving loop would: two device buffer sets
    (params, input batch, result copy) with the step captured once per set, the copies on their own
    stream, so step i+1's H2D and step i's D2H overlap step i's compute; every step still copies its own
    inputs and its own result."""
    ph = torch.from_numpy(W.params_h).pin_memory()
    xh = torch.from_numpy(W.x_h).to(torch.bfloat16).pin_memory()
    res = W.result()
    s = torch.cuda.current_stream()
    n = max(1, args.steps)
    has_x = bool(W.ins)
    P = [W.params, torch.empty_like(W.params)]
    X = [W.ins[0], torch.empty_like(W.ins[0])] if has_x else [None, None]
    Y = [torch.empty_like(res), torch.empty_like(res)]
    yh = [torch.empty(res.shape, dtype=res.dtype).pin_memory() for _ in range(2)]
    p0, x0 = W.params, (W.ins[0] if has_x else None)

    def use(b):
        W.params = P[b]
        if has_x:
            W.ins[0] = X[b]

    def body(b):
        W.construct()
        if W.sharded:
            W.gather(pg)
        W.forward()
        Y[b].copy_(res)
    steps = []
    for b in range(2):
        use(b)
        if graphs_ok and not W.sharded:
            g = capture(torch, lambda b=b: body(b))
            steps.append(g.replay)
        elif graphs_ok:
            gA = capture(torch, W.construct)
            gB = capture(torch, lambda b=b: (W.forward(), Y[b].copy_(res)))
            steps.append(lambda gA=gA, gB=gB: (gA.replay(), W.gather(pg), gB.replay()))
        else:
            steps.append(lambda b=b: (use(b), body(b)))
    use(0)
    torch.cuda.synchronize()
    c = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def loop(k):
        c.wait_stream(s)
        with torch.cuda.stream(c):                    # inputs of step 0
            P[0].copy_(ph, non_blocking=True)
            if has_x:
                X[0].copy_(xh, non_blocking=True)
            ev_in[0].record(c)
        for i in range(k):
            b = i % 2
            if i + 1 < k:                             # prefetch step i+1's inputs into the other set
                with torch.cuda.stream(c):
                    if i >= 1:
                        c.wait_event(ev_done[1 - b])  # step i-1 has finished reading that set
                    P[1 - b].copy_(ph, non_blocking=True)
                    if has_x:
                        X[1 - b].copy_(xh, non_blocking=True)
                    ev_in[1 - b].record(c)
            s.wait_event(ev_in[b])
            if i >= 2:
                s.wait_event(ev_out[b])               # Y[b] of step i-2 has reached the host
            steps[b]()
            ev_done[b].record(s)
            with torch.cuda.stream(c):                # D2H of step i's result
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
    W.params = p0
    if has_x:
        W.ins[0] = x0
    ms = t0.elapsed_time(t1) / n
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": len(W.layers) / (ms * 1e-3), "unit": "layers/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(ph.numel() * 4 + (xh.numel() * 2 if has_x else 0)),
            "d2h_bytes_per_step": int(Y[0].numel() * Y[0].element_size()),
            "launch": ("CUDA graph(s) per step and buffer set; H2D of step i+1 and D2H of step i on a copy stream "
                       "overlapping step i's compute (two buffer sets)" if graphs_ok else "eager")}


# ------------------------------------------------------------------ oracle (CPU) legs
def _threads():
    n = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(n)
    except Exception:
        pass
    return n


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


class OracleSampler:
    """The float64 oracle on a bounded sample of the workload.  Each sample is a window of w consecutive
    layers (rotating through the network): the oracle construction of ALL their matrices (power prescale,
    T = 12 Bjorck, BCOP / RKO / AOC composition) and the forward of ONE image through each of them at the
    layer's own input size.  The full step (construction + batch forward) is estimated per sampled layer as
    t_construct + batch * t_forward(1 image): that factor is the only extrapolation, and it is labelled."""

    def __init__(self, cfg_id, window):
        from synth import configs
        self.cfg_id = cfg_id
        self.layers = configs.CONFIGS[cfg_id]()
        self.batch = configs.BATCH[cfg_id]
        self.window = len(self.layers) if window <= 0 else min(window, len(self.layers))
        self.pos = 0
        self.reset()

    def reset(self):
        self.layer_s, self.sample_s, self.samples, self.layers_done = 0.0, [], 0, 0

    def sample(self):
        import oracle as O
        from synth import gen
        from tests.helpers import oracle_layer
        t_all = time.perf_counter()
        t_equiv = 0.0
        for j in range(self.window):
            l = (self.pos + j) % len(self.layers)
            d = self.layers[l]
            OL = oracle_layer(d)
            mats = []
            for g in range(OL.g):
                for i, M in enumerate(O.layer_matrices(OL)):
                    mats.append(gen.param_matrix(M.m, M.n, (self.cfg_id, l, g, i, gen.ROLE_ID[M.role])))
            t0 = time.perf_counter()
            ortho, _ = O.orthogonalize([A.astype(np.float64) for A in mats], T=12, beta=0.5, prescale="power", P=3)
            nm = len(O.layer_matrices(OL))
            K = O.layer_kernel(OL, [ortho[g * nm:(g + 1) * nm] for g in range(OL.g)])
            t1 = time.perf_counter()
            H = d["H"]
            x = gen.activations((1, d["c_in"], H, H), (self.cfg_id, 0, l, 0, gen.ROLE_ID["x"])).astype(np.float64)
            if d.get("kind") == "convT":
                O.conv_transpose2d(x, K, H * d["s"], H * d["s"], s=OL.s, d=OL.d, g=OL.g, mode=OL.padding_mode)
            else:
                O.conv2d(x, K, s=OL.s, d=OL.d, g=OL.g, mode=OL.padding_mode)
            t2 = time.perf_counter()
            t_equiv += (t1 - t0) + self.batch * (t2 - t1)
        self.pos = (self.pos + self.window) % len(self.layers)
        wall = time.perf_counter() - t_all
        self.layer_s += t_equiv
        self.layers_done += self.window
        self.sample_s.append(wall)
        self.samples += 1
        return wall

    def value(self):
        """layers/s of the full step over the sampled layers (construction measured; forward measured on
        one image and scaled to the batch)."""
        return self.layers_done / self.layer_s

    def describe(self):
        return (f"config {self.cfg_id}: {self.samples} samples of {self.window} consecutive layer(s), rotating: "
                f"float64 oracle construction of all their matrices (T=12) measured + forward of 1 image per "
                f"layer measured and x{self.batch} for the batch (the only extrapolation); "
                f"{self.layers_done} layer-samples of {len(self.layers)} layers")


def cpu_baseline(cfg_id, budget_s=20.0):
    cores = _threads()
    S = OracleSampler(cfg_id, window=1)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s and S.layers_done < 2 * len(S.layers):
        S.sample()
    return {"value": S.value(), "unit": "layers/s", "cores": cores, "kind": "oracle", "sample": S.describe(),
            "cpu": _cpu_model(), "wall_s": round(time.perf_counter() - t0, 2)}


def reference(args):
    """The oracle as the reference arm (tier framing: the CPU float64 oracle), rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import configs
    cores = _threads()
    cfg = args.config if args.config in configs.CONFIGS else 3
    S = OracleSampler(cfg, window=args.ref_window)
    for _ in range(min(args.warmup, 1)):
        S.sample()
    S.reset()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        S.sample()
    wall = time.perf_counter() - t0
    v = S.value()
    out = {"metric": METRIC, "value": v, "unit": "layers/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": configs.NAMES[cfg], "global_batch": configs.BATCH[cfg]},
           "step_is": "one bounded oracle sample; ms_per_step is its measured wall time",
           "extrapolation": f"value = sampled layers / sum over them of (construction + {configs.BATCH[cfg]} x "
                            f"one-image forward); equivalent full-step time {1e3 * len(S.layers) / v:.0f} ms",
           "wall_s": round(wall, 2),
           "cpu_baseline": {"value": v, "unit": "layers/s", "cores": cores, "kind": "oracle", "sample": S.describe(),
                            "cpu": _cpu_model()},
           "e2e": {"value": v, "unit": "layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def relaunch(args):
    """--gpus N > 1 without a torch.distributed environment: start N ranks (one per GPU) ourselves."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=2048, help="config 5: matrix size")
    ap.add_argument("--mats", type=int, default=64, help="config 5: number of n x n matrices")
    ap.add_argument("--compute", default="bf16", choices=["f32", "bf16", "bf16x3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying CUDA graphs")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-window", type=int, default=0,
                    help="reference arm: layers per oracle sample (0: the whole network per step)")
    ap.add_argument("--construct", default="sharded", choices=["sharded", "replicated"],
                    help="N > 1: shard construction by (layer, group) unit + all-gather, or replicate it")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
