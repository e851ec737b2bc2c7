"""One-shot vs one-iteration-per-call streaming ADMM: first differing iteration."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem, run_admm
import cnmf_oracle as O
a = O.dense_lowrank(1500, 900, 20, 0.01, seed=2).astype(np.float32)
A = DeviceMatrix(torch.from_numpy(a).cuda())
cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), 1500, 900)
left, right, core = compressed_problem(A, cfg)
run = lambda **kw: run_admm(core, left.panel, 1500, right.panel, 900, cfg, 20, **kw)
os.environ["CNMF_ADMM_STREAM"] = "1"
for n in (1, 2, 3, 5, 30):
    u0, v0, i0, t0 = run(max_iter=n, tol=0.0)
    u0b, v0b, _, t0b = run(max_iter=n, tol=0.0)
    u1, v1, i1, t1 = run(max_iter=n, tol=0.0, on_iteration=lambda *a: None)
    print(n, "oneshot repeat", (u0 - u0b).abs().max().item(), (v0 - v0b).abs().max().item(),
          "resume", (u0 - u1).abs().max().item(), (v0 - v1).abs().max().item(), i0, i1,
          np.abs(np.array(t0) - np.array(t1)).max())
sc = run(max_iter=200, tol=0.0)
os.environ.pop("CNMF_ADMM_STREAM")
for tol in (30, 10, 3, 1, 0.3, 0.1, 0.03):
    os.environ["CNMF_ADMM_STREAM"] = "1"
    a1 = run(max_iter=200, tol=tol)[2]
    os.environ.pop("CNMF_ADMM_STREAM")
    a2 = run(max_iter=200, tol=tol)[2]
    print("tol", tol, "stream", a1, "persistent", a2)
