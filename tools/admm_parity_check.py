import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import paper_1505_04650_b200 as C
from paper_1505_04650_b200 import _lib
import cnmf_oracle as O
a = O.dense_lowrank(2000, 1000, 20, 0.01, seed=0).astype(np.float32)
cfg = C.CompressionConfig(r=20, r_ov=10, w=4, seed=5)
ref = O.admm(a, 20, cfg=O.Config(20, 10, 4, 5), max_iter=500, tol=1e-4)
print("ref", ref.iterations, ref.rel_error)
for impl in (1, 0, 1):
    _lib.load().cnmf_set_pass_impl(impl)
    fp = C.nmf_admm(a, 20, cfg=cfg, max_iter=500, tol=1e-4)
    print("impl", impl, fp.iterations, fp.rel_error, abs(fp.rel_error - ref.rel_error) / ref.rel_error)
