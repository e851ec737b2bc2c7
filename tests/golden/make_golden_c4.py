"""Generate configs[4]-shaped range-finder fixtures (S = 64 panels) by
running the REFERENCE package itself (importable only in the build
container):

    python tests/golden/make_golden_c4.py

Writes ``tests/golden/reference_c4.npz``: for A = max(X Y + 0.01 N, 0) with
X ~ U[0, 1] (m x 50), Y 70 % zeros else U[0, 1] (50 x n) -- BASELINE.json
configs[4]'s distributions at reduced size -- and r = 50, r_ov = 10 (s = 60),
q = 4: the reference's ``structured_compress(..., reorthogonalize=True)``
column basis (fp32-rounded) and its own sensitivity band (projector distance
between its basis for A and for A * (1 + 2^-24 xi), three seeded xi). The
matrices are regenerated from the numpy seeds by the test.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_c4.npz")


def classical_config4(m, n, seed):
    """configs[4] generator at reduced size, fp32-rounded."""
    g = np.random.default_rng(seed)
    x = g.uniform(size=(m, 50))
    y = g.uniform(size=(50, n))
    y *= g.uniform(size=(50, n)) >= 0.7
    a = np.maximum(x @ y + 0.01 * g.standard_normal((m, n)), 0.0)
    return a.astype(np.float32).astype(np.float64)


def perturbed(a, k):
    xi = np.random.default_rng(7000 + k).standard_normal(a.shape)
    return a * (1.0 + 2.0 ** -24 * xi)


def proj_dist(q1, q2):
    return float(np.linalg.norm(q2 - q1 @ (q1.T @ q2), 2))


def main():
    sys.path.insert(0, REF)
    import cnmf
    from cnmf import CompressionConfig

    fx = {}
    for (m, n) in ((4000, 2000), (12000, 6000)):
        a = classical_config4(m, n, seed=13)
        cfg = CompressionConfig(r=50, r_ov=10, w=4, seed=3)
        q = cnmf.structured_compress(a, cfg, reorthogonalize=True).q_dense()
        band = [proj_dist(q, cnmf.structured_compress(perturbed(a, k), cfg, reorthogonalize=True).q_dense())
                for k in range(3)]
        key = f"c4_{m}x{n}"
        fx[key + "_q"] = q.astype(np.float32)
        fx[key + "_band"] = np.array(band)
        print(key, "band", band, flush=True)
    np.savez_compressed(OUT, **fx)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
