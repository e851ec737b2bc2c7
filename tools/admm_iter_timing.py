"""Streaming-ADMM time per iteration vs problem height: with tiny m, n the
row sweep is negligible and the time is the core step's."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import zeros
from paper_1505_04650_b200.nmf import run_admm

r, s = 50, 60
for m, n in ((2000, 1000), (20000, 10000), (200_000, 100_000)):
    g = torch.Generator(device="cuda").manual_seed(0)
    lp = zeros((m, 64))
    rp = zeros((n, 64))
    lp[:, :s] = torch.linalg.qr(torch.randn(m, s, device="cuda", generator=g))[0]
    rp[:, :s] = torch.linalg.qr(torch.randn(n, s, device="cuda", generator=g))[0]
    core = torch.rand(s, s, device="cuda", dtype=torch.float64, generator=g) * 100
    cfg = C.CompressionConfig(r=r, r_ov=10, w=4, seed=1)
    run_admm(core, lp, m, rp, n, cfg, r, max_iter=3, tol=0.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run_admm(core, lp, m, rp, n, cfg, r, max_iter=50, tol=0.0)
    e1.record()
    torch.cuda.synchronize()
    print(f"m={m} n={n}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per iteration", flush=True)
