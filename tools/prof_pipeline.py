"""One configs[1] pipeline step (for ncu launch lists): compress L and R,
core, ADMM (100 iterations, tol=0), relative error."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix

M, N, R = 10000, 5000, 20
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.addmm(0.01 * torch.randn(M, N, device="cuda", generator=g), torch.rand(M, R, device="cuda", generator=g),
                torch.rand(R, N, device="cuda", generator=g)).clamp_(min=0)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
fp = C.nmf_admm(a, R, cfg=C.CompressionConfig(r=R, r_ov=10, w=4, seed=5), max_iter=iters, tol=0.0)
torch.cuda.synchronize()
print("rel_error", fp.rel_error, "iterations", fp.iterations)
