import sys; sys.path.insert(0, "/root/repo")
import torch, paper_2601_13776_b200 as orth
from synth import configs, gen
layers = configs.cfg5(2048)
plan = orth.Plan(layers, 0, compute="bf16")
params = torch.zeros(plan.params_numel, device="cuda")
for i, m in enumerate(plan.matrices):
    params[m["off"]: m["off"] + m["m"] * m["n"]] = gen.param_matrix_torch(m["m"], m["n"], (5, m["layer"], m["group"], i, gen.ROLE_ID[m["role"]]), torch, torch.device("cuda")).ravel()
o = torch.zeros_like(params)
for _ in range(2): plan.orthogonalize(params, o)
torch.cuda.synchronize()
