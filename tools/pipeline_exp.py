"""Experiment: overlap the construction of the deep layers with the forward of the early ones (cfg3).
Splits the network into two plans at layer `a`; times (1) one plan, serial; (2) two plans, serial;
(3) two plans with the deep plan's construction on a second stream, overlapping the early convs.
All as CUDA graphs, CUDA events, L2 flushed between steps.  python tools/pipeline_exp.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs, gen  # noqa: E402


class Part:
    def __init__(self, layers, l0, N, x_in, cfg_id=3):
        self.plan = plan = orth.Plan(layers, 0, compute="bf16", max_batch=N)
        params = np.zeros(plan.params_numel, np.float32)
        for i, m in enumerate(plan.matrices):
            A = gen.param_matrix(m["m"], m["n"], (cfg_id, m["layer"] + l0, m["group"], i, gen.ROLE_ID[m["role"]]))
            params[m["off"]: m["off"] + A.size] = A.ravel()
        self.params = torch.from_numpy(params).cuda()
        self.cache = torch.zeros(plan.cache_numel, device="cuda") + 0.1
        self.ortho = torch.zeros_like(self.params)
        self.kf = torch.zeros(plan.kf32_numel, device="cuda")
        self.kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
        self.ins, self.outs = [], []
        x = x_in
        for l, d in enumerate(layers):
            H = x.shape[1]
            Ho, _ = plan.out_hw(l, H, H)
            y = torch.empty(N, Ho, Ho, d["c_out"], device="cuda", dtype=torch.bfloat16)
            self.ins.append(x)
            self.outs.append(y)
            x = y
        self.kv = [plan.kernel_bf16(self.kb, l) for l in range(len(layers))]

    def construct(self):
        self.plan.orthogonalize(self.params, self.ortho, self.cache)
        self.plan.compose(self.ortho, self.kf, self.kb)

    def forward(self):
        for l in range(len(self.ins)):
            self.plan.conv_forward(l, self.kv[l], self.ins[l], self.outs[l])


def capture(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()   # warm
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return g


def timeit(g, reps=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 3):
        flush.fill_(i & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    layers = configs.cfg3()
    N = 256
    x = torch.from_numpy(gen.activations((N, 224, 224, 3), (3, 0, 0, 0, 1))).cuda().to(torch.bfloat16)
    whole = Part(layers, 0, N, x)

    def one():
        whole.construct()
        whole.forward()
    print("one plan, serial: %.3f ms" % timeit(capture(one)), flush=True)
    for a in (7, 15, 27):
        p0 = Part(layers[:a], 0, N, x)
        p1 = Part(layers[a:], a, N, p0.outs[-1])

        def serial():
            p0.construct()
            p0.forward()
            p1.construct()
            p1.forward()

        side = torch.cuda.Stream()

        def overlap():
            cur = torch.cuda.current_stream()
            p0.construct()
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                p1.construct()
            p0.forward()
            cur.wait_stream(side)
            p1.forward()
        print("split %d: two plans serial %.3f ms, overlapped %.3f ms" % (a, timeit(capture(serial)),
                                                                         timeit(capture(overlap))), flush=True)

        def c0():
            p0.construct()

        def c1():
            p1.construct()

        def f0():
            p0.forward()

        def f1():
            p1.forward()
        print("   parts: construct0 %.3f construct1 %.3f forward0 %.3f forward1 %.3f" % (
            timeit(capture(c0)), timeit(capture(c1)), timeit(capture(f0)), timeit(capture(f1))), flush=True)


if __name__ == "__main__":
    main()
