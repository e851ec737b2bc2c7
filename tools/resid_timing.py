"""Time the fused residual-norm pass (||A - XY||, ||A||) on a configs[1]-shaped A."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros

M, N, R = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10000, 5000, 20)))
a = torch.rand(M, N, device="cuda")
A = DeviceMatrix(a)
x = torch.rand(M, R, device="cuda", dtype=torch.float64)
yt = torch.rand(N, R, device="cuda", dtype=torch.float64)
res = zeros((2,), torch.float64)
f = lambda: _lib.call("cnmf_residual_norms", A.ptr, M, N, A.lda, x.data_ptr(), None, yt.data_ptr(), R, res.data_ptr(), stream())
for _ in range(3):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
ref = ((a.double() - x @ yt.t()) ** 2).sum().item(), (a.double() ** 2).sum().item()
print(f"residual pass {ms * 1e3:.1f} us, {4 * M * N / ms / 1e6:.0f} GB/s; rel diff {abs(res[0].item() - ref[0]) / ref[0]:.2e} {abs(res[1].item() - ref[1]) / ref[1]:.2e}")
