"""Run the row_mma micro (tools/micro/row_mma.so) inside a PyTorch process, after torch CUDA work and
after one call of the library's conv (the ROW layer): does the process context change tcgen05 rates?"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "row_mma.so"))
print("== before torch", flush=True)
lib.row_mma_main()
import torch  # noqa: E402
x = torch.randn(1 << 20, device="cuda")
torch.cuda.synchronize()
print("== after torch init", flush=True)
lib.row_mma_main()
import paper_2601_13776_b200 as orth  # noqa: E402
layer = dict(kind="conv", c_in=64, c_out=64, k=3, s=1, d=1, g=1, padding_mode="circular", grid=(56, 56))
plan = orth.Plan([layer], 0, max_batch=256)
kb = (torch.randn(64, 3, 3, 64, device="cuda") * 0.05).to(torch.bfloat16)
xx = torch.randn(256, 56, 56, 64, device="cuda").to(torch.bfloat16)
y = torch.empty_like(xx)
for _ in range(3):
    plan.conv_forward(0, kb, xx, y)
torch.cuda.synchronize()
print("== after library conv", flush=True)
lib.row_mma_main()
