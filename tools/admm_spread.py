import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
import cnmf_oracle as O
import paper_1505_04650_b200 as C
a = O.dense_lowrank(2000, 1000, 20, 0.01, seed=0).astype(np.float32)
cfg = C.CompressionConfig(r=20, r_ov=10, w=4, seed=5)
print([C.nmf_admm(a, 20, cfg=cfg, max_iter=500, tol=1e-4).rel_error for _ in range(5)])
