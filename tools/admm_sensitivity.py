"""Where does the device/oracle ADMM gap on a configs[1]-shaped problem come
from? Device bases (tensor-core and FFMA passes) vs the oracle's, and the
oracle ADMM re-run on the device bases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from dataclasses import replace

import numpy as np

import cnmf_oracle as O
import paper_1505_04650_b200 as C
from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem

m, n = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (2000, 1000)))
a32 = O.dense_lowrank(m, n, 20, 0.01, seed=0).astype(np.float32)
a = a32.astype(np.float64)
ocfg = O.adjust(O.Config(20, 10, 4, 5), m, n)
L, R = O.compressed_bases(a, ocfg, True)
ref = O.admm(a, 20, cfg=O.Config(20, 10, 4, 5), max_iter=500, tol=1e-4, bases=(L, R))
print(f"oracle rel_error {ref.rel_error:.10f}")


def pd(q1, q2):
    return O.projector_distance(q1, q2)


for impl in (1, 0):
    _lib.load().cnmf_set_pass_impl(impl)
    cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), m, n)
    left, right, core = compressed_problem(DeviceMatrix(a32), cfg)
    Ld = left.Q
    Rd = right.Q.T  # s x n
    sig = slice(0, 20)
    print(f"impl={'tc' if impl else 'ffma'} pd(L)={pd(L, Ld):.3e} pd(R)={pd(R.T, Rd.T):.3e} "
          f"pd(L[:, :20])={pd(L[:, sig], Ld[:, sig]):.3e}")
    core_o = (L.T @ a) @ R.T
    core_dd = (Ld.T @ a) @ Rd.T
    print(f"   core(dev bases, fp64) vs device core: {np.abs(core.cpu().numpy() - core_dd).max() / np.abs(core_dd).max():.3e}")
    o2 = O.admm(a, 20, cfg=O.Config(20, 10, 4, 5), max_iter=500, tol=1e-4, bases=(Ld, Rd))
    print(f"   oracle ADMM on device bases: rel_error {o2.rel_error:.10f} dev {abs(o2.rel_error - ref.rel_error) / ref.rel_error:.3e}")
    fp = C.nmf_admm(a32, 20, cfg=C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), max_iter=500, tol=1e-4)
    print(f"   device ADMM: rel_error {fp.rel_error:.10f} dev {abs(fp.rel_error - ref.rel_error) / ref.rel_error:.3e}")
