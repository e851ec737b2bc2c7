"""Tensor-core pass vs fp64 reference at a given shape: max relative error
per pass, and run-to-run bitwise equality."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros

M, N, S = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10000, 5000, 32)))
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.rand(M, N, device="cuda", generator=g)
A = DeviceMatrix(a)
X = torch.randn(N, S, device="cuda", generator=g)
W = torch.randn(M, S, device="cuda", generator=g)
yref = a.double() @ X.double()
zref = a.double().t() @ W.double()
for name, fn, ref, rows in (("fwd", lambda o: lib.cnmf_pass_forward(A.ptr, M, N, A.lda, X.data_ptr(), S, o.data_ptr(), stream()), yref, M),
                            ("trn", lambda o: lib.cnmf_pass_transpose(A.ptr, M, N, A.lda, W.data_ptr(), S, o.data_ptr(), stream()), zref, N)):
    outs = []
    for _ in range(3):
        o = zeros((rows, S))
        fn(o)
        torch.cuda.synchronize()
        outs.append(o.double())
    err = ((outs[0] - ref).abs() / ref.abs().max()).max(dim=1).values
    bad = (err > 1e-5).nonzero().flatten()
    print(f"{name} {M}x{N} S={S}: max rel err {err.max().item():.2e}, bad rows {bad.numel()} "
          f"(first {bad[:8].tolist()}), bitwise repeat {all(torch.equal(outs[0], o) for o in outs[1:])}", flush=True)
