"""XRAY on a configs[3]-shaped reduced matrix (no profiler): the ncu target."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1505_04650_b200 as C
g = np.random.default_rng(0)
s, n, r = 60, int(os.environ.get("XN", "200000")), int(os.environ.get("XR", "50"))
w0 = np.abs(g.standard_normal((s, 50)))
h = np.zeros((50, n)); h[:, :50] = np.eye(50); h[:, 50:] = g.dirichlet(np.ones(50), size=n - 50).T
h = h[:, g.permutation(n)]
red_d = torch.from_numpy(w0 @ h + 0.01 * g.standard_normal((s, n))).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
picks = C.select_columns_xray(red_d, r)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0, "picks", [int(x) for x in picks[:8]])
