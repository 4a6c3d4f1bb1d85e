import sys, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2601_13776_b200 as orth
from synth import configs
from tests.helpers import pack_params
L = configs.cfg2()
for name, sub in [("all", L), ("early0-8", L[:9]), ("late9-11", L[9:]), ("early0-9", L[:10]), ("late10-11", L[10:])]:
    plan = orth.Plan(sub, 0, compute="bf16")
    params, _ = pack_params(plan, 2)
    p = torch.from_numpy(params).cuda(); o = torch.zeros_like(p)
    kf = torch.zeros(plan.kf32_numel, device="cuda"); kb = torch.zeros(plan.kbf16_numel, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        plan.orthogonalize(p, o); plan.compose(o, kf, kb)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_o = t_c = 0
    for _ in range(10):
        e[0].record(); plan.orthogonalize(p, o); e[1].record(); plan.compose(o, kf, kb); e[2].record()
        torch.cuda.synchronize(); t_o += e[0].elapsed_time(e[1]); t_c += e[1].elapsed_time(e[2])
    print(f"{name:10s} matrices {plan.n_matrices:3d}: orth {t_o/10*1e3:.0f} us, compose {t_c/10*1e3:.0f} us")
