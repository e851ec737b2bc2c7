"""Time the compressed problem (both range finders + core) on configs[1]
(CUDA graph replay and eager), and compare the paired bases against the
single-chain ones (projector distance)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_04650_b200 as C
from paper_1505_04650_b200.compress import _compress
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem
from paper_1505_04650_b200.rng import child_seed
from dataclasses import replace

M, N, R = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10000, 5000, 20)))
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(M, R, device="cuda", generator=g)
y = torch.rand(R, N, device="cuda", generator=g)
a = torch.addmm(0.01 * torch.randn(M, N, device="cuda", generator=g), x, y).clamp_(min=0.0)
A = DeviceMatrix(a)
cfg = C.adjust_config(C.CompressionConfig(r=R, r_ov=10, w=4, seed=5), M, N)
s = cfg.basis_cols
for graph in (True, False):
    for _ in range(3):
        compressed_problem(A, cfg, graph=graph)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        left, right, core = compressed_problem(A, cfg, check=False, graph=graph)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"compressed problem ({'graph' if graph else 'eager'}): {ms:.3f} ms -> {19 * M * N * 4 / ms / 1e6:.0f} GB/s per pass")
lb, _ = _compress(A, replace(cfg, seed=child_seed(cfg.seed, "left-basis")), 0)
rb, _ = _compress(A, replace(cfg, seed=child_seed(cfg.seed, "right-basis")), 1)


def pdist(p, q):
    p = p[:, :s].double()
    q = q[:, :s].double()
    return torch.linalg.matrix_norm(p @ p.t() - q @ q.t(), ord=2).item() if p.shape[0] <= 6000 else \
        torch.linalg.svdvals(torch.cat([p, q], 1)).max().item()


left, right, core = compressed_problem(A, cfg, graph=False)
for nm, p, q in (("left", left.panel, lb.panel), ("right", right.panel, rb.panel)):
    pp, qq = p[:, :s].double(), q[:, :s].double()
    # ||P P^T - Q Q^T||_2 = sin of the largest principal angle
    sv = torch.linalg.svdvals(pp.t() @ qq).clamp(max=1.0)
    print(nm, "projector distance vs single chain:", torch.sqrt(1 - sv.min() ** 2).item(),
          "orthonormality", (pp.t() @ pp - torch.eye(s, device="cuda", dtype=torch.float64)).abs().max().item())
