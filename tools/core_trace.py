"""Phase durations of the streaming ADMM core step (needs a library built
with -DCNMF_CORE_TRACE, e.g. CNMF_LIB_PATH=varlibs/coretrace.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1505_04650_b200 as C
from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import zeros
from paper_1505_04650_b200.nmf import run_admm

m, n, r, s = 200_000, 100_000, 50, 60
g = torch.Generator(device="cuda").manual_seed(0)
lp = zeros((m, 64))
rp = zeros((n, 64))
lp[:, :s] = torch.linalg.qr(torch.randn(m, s, device="cuda", generator=g))[0]
rp[:, :s] = torch.linalg.qr(torch.randn(n, s, device="cuda", generator=g))[0]
core = torch.rand(s, s, device="cuda", dtype=torch.float64, generator=g) * 100
cfg = C.CompressionConfig(r=r, r_ov=10, w=4, seed=1)
lib = _lib.load()
fn = lib.cnmf_debug_core_trace
for it in (4, 5, 6):
    run_admm(core, lp, m, rp, n, cfg, r, max_iter=it, tol=0.0)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 16)()
    fn(buf)
    t = list(buf)
    names = ["load", "dual proj", "kkt", "M, rhs", "inverse 1", "xc, M2, rhs2", "inverse 2", "yc"]
    print(it, " | ".join(f"{nm} {(t[i + 1] - t[i]) / 1.9e3:.1f}us" for i, nm in enumerate(names) if t[i + 1] > t[i]))
