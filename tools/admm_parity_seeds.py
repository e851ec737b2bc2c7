"""Device vs oracle final NMF relative error over several seeds of the
configs[1]-shaped parity case, next to the oracle's own sensitivity to an
fp32-rounding-sized perturbation of A (how far the reference itself moves)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np

import cnmf_oracle as O
import paper_1505_04650_b200 as C

m, n = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (2000, 1000)))
for seed in range(int(os.environ.get("SEEDS", 6))):
    a = O.dense_lowrank(m, n, 20, 0.01, seed=seed).astype(np.float32)
    cfg = C.CompressionConfig(r=20, r_ov=10, w=4, seed=5 + seed)
    fp = C.nmf_admm(a, 20, cfg=cfg, max_iter=int(os.environ.get("ITERS", 500)), tol=1e-4)
    ref = O.admm(a, 20, cfg=O.Config(20, 10, 4, 5 + seed), max_iter=int(os.environ.get("ITERS", 500)), tol=1e-4)
    g = np.random.default_rng(100 + seed)
    ap = a.astype(np.float64) * (1.0 + 6e-8 * g.standard_normal(a.shape))
    ref2 = O.admm(ap, 20, cfg=O.Config(20, 10, 4, 5 + seed), max_iter=int(os.environ.get("ITERS", 500)), tol=1e-4)
    d = (fp.rel_error - ref.rel_error) / ref.rel_error
    d2 = (ref2.rel_error - ref.rel_error) / ref.rel_error
    print(f"seed {seed}: device {fp.rel_error:.8f} oracle {ref.rel_error:.8f} dev {d:+.2e} | "
          f"oracle on A(1+6e-8 N(0,1)): dev {d2:+.2e} | iters {fp.iterations} {ref.iterations}", flush=True)
