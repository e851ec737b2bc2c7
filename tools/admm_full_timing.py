"""Time nmf_admm(compressed=False) per iteration on configs[1]'s matrix
(10000 x 5000, r = 20): two passes over A plus three row kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_04650_b200 as C

m, n, r = 10000, 5000, 20
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(m, r, device="cuda", generator=g)
y = torch.rand(r, n, device="cuda", generator=g)
a = torch.addmm(0.01 * torch.randn(m, n, device="cuda", generator=g), x, y).clamp_(min=0.0)
cfg = C.CompressionConfig(r=r, r_ov=10, w=4, seed=5)
for iters in (10, 110):
    C.nmf_admm(a, r, compressed=False, cfg=cfg, max_iter=iters, tol=0.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = C.nmf_admm(a, r, compressed=False, cfg=cfg, max_iter=iters, tol=0.0)
    torch.cuda.synchronize()
    print(f"uncompressed ADMM {iters} iterations: {1e3 * (time.perf_counter() - t0):.2f} ms, rel error {res.rel_error:.5f}")
