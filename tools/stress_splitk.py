"""Repeat passes on split-K shapes; report launches that differ from the first
(bit-for-bit) and the rows that differ."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros
lib = _lib.load()
for (m, n, S) in [(12000, 6000, 64), (3000, 4000, 64), (10000, 5000, 32), (12000, 6000, 32)]:
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.rand(m, n, device="cuda", generator=g)
    A = DeviceMatrix(a)
    x = torch.randn(n, S, device="cuda", generator=g)
    w = torch.randn(m, S, device="cuda", generator=g)
    for name, P, fn in (("fwd", m, lambda o: lib.cnmf_pass_forward(A.ptr, m, n, A.lda, x.data_ptr(), S, o, stream())),
                        ("trn", n, lambda o: lib.cnmf_pass_transpose(A.ptr, m, n, A.lda, w.data_ptr(), S, o, stream()))):
        ref = zeros((P, S)); fn(ref.data_ptr()); torch.cuda.synchronize()
        exact = (a.double() @ x.double()) if name == "fwd" else (a.double().t() @ w.double())
        print("  ref error", ((ref.double() - exact).abs().max() / exact.abs().max()).item())
        bad = 0; rows = set()
        for it in range(200):
            o = zeros((P, S)); fn(o.data_ptr()); torch.cuda.synchronize()
            if not torch.equal(o, ref):
                bad += 1
                d = (o != ref).any(1).nonzero().flatten().tolist()
                rows.update(d[:5])
                if bad <= 3:
                    print("  bad launch", it, "err vs exact", ((o.double() - exact).abs().max() / exact.abs().max()).item(),
                          "ntiles", len(set(r // 256 for r in d)), "tiles", sorted(set(r // 256 for r in d))[:10], flush=True)
        print(m, n, S, name, "mismatching launches", bad, "rows", sorted(rows)[:20], flush=True)
