"""Forward / transpose / paired passes against torch fp64 on split-K shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros
lib = _lib.load()
for (m, n, S) in [(12000, 6000, 64), (12000, 6000, 32), (4000, 2000, 64), (3000, 4000, 64), (10000, 5000, 32)]:
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.rand(m, n, device="cuda", generator=g)
    A = DeviceMatrix(a)
    x = torch.randn(n, S, device="cuda", generator=g)
    w = torch.randn(m, S, device="cuda", generator=g)
    y, z, y2, z2 = zeros((m, S)), zeros((n, S)), zeros((m, S)), zeros((n, S))
    lib.cnmf_pass_forward(A.ptr, m, n, A.lda, x.data_ptr(), S, y.data_ptr(), stream())
    lib.cnmf_pass_transpose(A.ptr, m, n, A.lda, w.data_ptr(), S, z.data_ptr(), stream())
    lib.cnmf_pass_pair(A.ptr, m, n, A.lda, x.data_ptr(), y2.data_ptr(), w.data_ptr(), z2.data_ptr(), S, stream())
    torch.cuda.synchronize()
    yr, zr = a.double() @ x.double(), a.double().t() @ w.double()
    e = lambda u, r: ((u.double() - r).abs().max() / r.abs().max()).item()
    bad = lambda u, r: int(((u.double() - r).abs() > 1e-4 * r.abs().max()).any(1).sum().item())
    print(m, n, S, "fwd", e(y, yr), bad(y, yr), "trn", e(z, zr), bad(z, zr), "pair", e(y2, yr), bad(y2, yr), e(z2, zr), bad(z2, zr), flush=True)
