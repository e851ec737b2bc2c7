"""Streaming ADMM at the configs[4] size (m=200000, n=100000, s=60, r=50), 6 iterations: the ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import zeros
from paper_1505_04650_b200.nmf import run_admm
m, n, r, s = 200_000, 100_000, 50, 60
g = torch.Generator(device="cuda").manual_seed(0)
lp = zeros((m, 64)); rp = zeros((n, 64))
lp[:, :s] = torch.linalg.qr(torch.randn(m, s, device="cuda", generator=g))[0]
rp[:, :s] = torch.linalg.qr(torch.randn(n, s, device="cuda", generator=g))[0]
core = torch.rand(s, s, device="cuda", dtype=torch.float64, generator=g) * 100
cfg = C.CompressionConfig(r=r, r_ov=10, w=4, seed=1)
run_admm(core, lp, m, rp, n, cfg, r, max_iter=6, tol=0.0)
torch.cuda.synchronize()
print("ok")
