"""How sensitive is the REFERENCE's own configs[2] outcome (oracle port, fp64)
to fp32-rounding-sized perturbations of A? For each seed: the oracle on A,
then on A * (1 + 2^-24 xi) for a few seeded xi ~ N(0, 1) (a perturbation
the size of one fp32 rounding of A). Reports, per run, the SPA picks and
whether the NNLS right factor trips the reference's exchange cap
(ConvergenceError) or returns.

usage: python tools/snmf_config2_sensitivity.py [m] [n_perturbations]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import cnmf_oracle as O

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
npert = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for seed in (1, 2):
    a, truth = O.near_separable(m, 200, 20, 0.5, 0.005, seed=seed)
    a = a.astype(np.float32).astype(np.float64)
    for p in range(npert + 1):
        if p == 0:
            ap = a
        else:
            xi = np.random.default_rng(1000 + p).standard_normal(a.shape)
            ap = a * (1.0 + 2.0 ** -24 * xi)
        t = time.time()
        cfg = O.adjust(O.Config(20, 10, 2, 7), *ap.shape)
        q = O.range_basis(ap, cfg)
        red = q.T @ ap
        picks = O.spa(red, 20)
        try:
            O.nnls(red[:, picks], red, tol=1e-10)
            out = "NNLS returns"
        except O.OracleError as e:
            out = f"NNLS raises {e.kind}"
        print(f"m={m} seed={seed} perturbation={p}: {out}; picks = the true columns: "
              f"{sorted(picks.tolist()) == sorted(truth.tolist())}; order {picks[:6].tolist()} ({time.time() - t:.1f} s)",
              flush=True)
