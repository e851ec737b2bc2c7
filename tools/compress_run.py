"""Two eager compressed problems on configs[1] (for ncu captures of the
range-finder kernels: pass_tc, sweep_kernel, test-matrix kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem

g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(10000, 20, device="cuda", generator=g)
y = torch.rand(20, 5000, device="cuda", generator=g)
a = torch.addmm(0.01 * torch.randn(10000, 5000, device="cuda", generator=g), x, y).clamp_(min=0.0)
A = DeviceMatrix(a)
cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), 10000, 5000)
for _ in range(2):
    compressed_problem(A, cfg, graph=False)
torch.cuda.synchronize()
print("ok")
