"""Run-to-run spread of the device ADMM on one fixed compressed problem
(the atomics reduce in a nondeterministic order), per scheduling mode, and
the step-by-step resume path (on_iteration) against the single launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch
import cnmf_oracle as O
import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem, run_admm

m, n, r = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (2000, 1001, 20)))
a32 = O.dense_lowrank(m, n, r, 0.01, seed=0).astype(np.float32)
A = DeviceMatrix(torch.from_numpy(a32).cuda())
cfg = C.adjust_config(C.CompressionConfig(r=r, r_ov=10, w=4, seed=5), m, n)
left, right, core = compressed_problem(A, cfg)
def run(**kw):
    u, vt, it, tr = run_admm(core, left.panel, m, right.panel, n, cfg, r, max_iter=int(os.environ.get("ITERS", 500)),
                             tol=1e-4, **kw)
    torch.cuda.synchronize()
    a = torch.from_numpy(a32).cuda().double()
    rel = float(torch.linalg.norm(a - u @ vt.t()) / torch.linalg.norm(a))
    return u.cpu().numpy(), it, rel, tr
for mode in os.environ.get("MODES", "1,0").split(","):
    os.environ["CNMF_ADMM_SPEC"] = mode
    outs = [run() for _ in range(int(os.environ.get("REPS", 6)))]
    u0 = outs[0][0]
    print(f"spec={mode} iters {[o[1] for o in outs]} rel {[f'{o[2]:.10f}' for o in outs]} "
          f"max|U-U0| {max(float(np.abs(o[0] - u0).max()) for o in outs):.3e}")
    if os.environ.get("STEP"):
        seen = []
        o = run(on_iteration=lambda k, *a: seen.append(k))
        print(f"  stepwise: iters {o[1]} rel {o[2]:.10f} callbacks {len(seen)} trace equal "
              f"{np.allclose(o[3], outs[0][3], rtol=1e-6)}")
