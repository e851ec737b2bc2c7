"""Forward-pass error vs fp64 as a function of K, tensor-core vs FFMA."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros

lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
M, S = 4096, int(os.environ.get("PA_S", "32"))
for K in (256, 1024, 4096, 16384):
    a = torch.rand(M, K, device="cuda", generator=g)
    x = torch.randn(K, S, device="cuda", generator=g)
    ref = a.double() @ x.double()
    scale = (a.double().abs() @ x.double().abs())
    A = DeviceMatrix(a)
    line = f"K={K:6d}"
    for impl in (1, 0):
        lib.cnmf_set_pass_impl(impl)
        y = zeros((M, S))
        lib.cnmf_pass_forward(A.ptr, M, K, A.lda, x.data_ptr(), S, y.data_ptr(), stream())
        torch.cuda.synchronize()
        e = ((y.double() - ref) / scale)
        line += f" | {'tc' if impl else 'ffma'} max {e.abs().max().item():.2e} mean {e.mean().item():+.2e} rms {e.pow(2).mean().sqrt().item():.2e}"
    print(line, flush=True)
    # transpose pass: Z = A^T W, K = M rows
    w = torch.randn(M, S, device="cuda", generator=g)
    ref = a.double().t() @ w.double()
    scale = a.double().abs().t() @ w.double().abs()
    line = f"  T K={M:6d} P={K:6d}"
    for impl in (1, 0):
        lib.cnmf_set_pass_impl(impl)
        z = zeros((K, S))
        lib.cnmf_pass_transpose(A.ptr, M, K, A.lda, w.data_ptr(), S, z.data_ptr(), stream())
        torch.cuda.synchronize()
        e = ((z.double() - ref) / scale)
        line += f" | {'tc' if impl else 'ffma'} max {e.abs().max().item():.2e} mean {e.mean().item():+.2e} rms {e.pow(2).mean().sqrt().item():.2e}"
    print(line, flush=True)
