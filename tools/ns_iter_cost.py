"""Per-iteration cost of the tensor-core NS loop on a config (graph replay,
warm L2): time orthogonalize at several T and fit the slope."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs  # noqa: E402
from tests.helpers import pack_params  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
compute = sys.argv[2] if len(sys.argv) > 2 else "bf16"
layers = configs.CONFIGS[cfg]()
for T in (1, 2, 6, 12):
    for pi in (3, 1):
        plan = orth.Plan(layers, 0, compute=compute, ns_iters=T, power_iters=pi, polish_iters=min(2, T))
        params, _ = pack_params(plan, cfg)
        p = torch.from_numpy(params).cuda()
        o = torch.zeros_like(p)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                plan.orthogonalize(p, o)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            plan.orthogonalize(p, o)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        print(f"T={T:2d} power_iters={pi}  {a.elapsed_time(b) / 50 * 1000:8.1f} us", flush=True)
