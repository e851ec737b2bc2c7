"""One configs[1]-shaped two-sided compression (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem

M, N, R = 10000, 5000, 20
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.addmm(0.01 * torch.randn(M, N, device="cuda", generator=g), torch.rand(M, R, device="cuda", generator=g),
                torch.rand(R, N, device="cuda", generator=g)).clamp_(min=0)
A = DeviceMatrix(a)
cfg = C.adjust_config(C.CompressionConfig(r=R, r_ov=10, w=4, seed=5), M, N)
for _ in range(int(os.environ.get("REPS", "2"))):
    compressed_problem(A, cfg)
torch.cuda.synchronize()
print("ok")
