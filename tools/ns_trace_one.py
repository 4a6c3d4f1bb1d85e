"""NS flow trace of small plans (diagnostics build: ORTH_NVCC_FLAGS=-DORTH_NSP_TRACE, ORTH_NS_TRACE=1):
python tools/ns_trace_one.py {dense|cfg2|cfg3} -- prints the per-phase report of the largest matrices."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_13776_b200 as orth  # noqa: E402
from synth import configs  # noqa: E402
from tests.helpers import pack_params  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "dense"
if which == "dense":
    layers = [dict(kind="dense", c_in=512, c_out=1024, k=1, s=1, d=1, g=1, padding_mode="circular")]
elif which == "dense4":
    layers = [dict(kind="dense", c_in=512, c_out=1024, k=1, s=1, d=1, g=1, padding_mode="circular")] * 4
else:
    layers = configs.CONFIGS[int(which[-1])]()
plan = orth.Plan(layers, 0, compute="bf16")
params, _ = pack_params(plan, 2)
p = torch.from_numpy(params).cuda()
o = torch.zeros_like(p)
for _ in range(3):
    plan.orthogonalize(p, o)
torch.cuda.synchronize()
plan.check()
