"""Debug: streaming ADMM (CNMF_ADMM_STREAM=1) on a small problem, first iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_04650_b200 as C
from oracle import cnmf_oracle as O
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem, run_admm
a = O.dense_lowrank(2000, 1001, 20, 0.01, seed=0).astype(np.float32)
A = DeviceMatrix(torch.from_numpy(a).cuda())
cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), 2000, 1001)
left, right, core = compressed_problem(A, cfg)
for force in ("0", "1"):
    os.environ["CNMF_ADMM_STREAM"] = force
    for it in (1, 2, 3):
        u, vt, k, tr = run_admm(core, left.panel, 2000, right.panel, 1001, cfg, 20, max_iter=it, tol=0.0)
        torch.cuda.synchronize()
        print(force, it, k, float(u.abs().max()), float(vt.abs().max()), float(u.isnan().sum()), tr[:3])
