"""Generate the full-size parity fixtures by running the REFERENCE package
itself (importable only in the build container):

    python tests/golden/make_golden_large.py

Writes ``tests/golden/reference_large.npz``. The matrices are NOT stored: the
tests regenerate them on the GPU box from the same numpy seeds (numpy's
default_rng streams are platform independent), so only bases, picks and
scalars are committed.

Contents
* configs[1]-shaped range finder (A = max(X Y + 0.01 N, 0), X, Y ~ U[0, 1],
  r = 20, s = 30, q = 4) at 2000 x 1000 and 10000 x 5000: the reference's
  ``structured_compress(..., reorthogonalize=True)`` basis (fp32-rounded),
  the reference's OWN sensitivity band -- the projector distance between its
  basis for A and for A * (1 + 2^-24 xi) (one fp32 rounding of A), three
  seeded xi -- and, for the record, the distance to the stock
  ``reorthogonalize=False`` basis and both compression errors.
* configs[2]-shaped tall SNMF (2,000,000 x 200, r = 20, Dirichlet(0.5), noise
  0.005, q = 2, SPA) for seeds 1 and 2: the reference's SPA picks on its
  reduced matrix, and whether its NNLS right factor (tol 1e-10) returns or
  trips the exchange cap -- for A and for three 2^-24 perturbations of A.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_large.npz")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))


def dense_config1(m, n, seed):
    """configs[1] generator (oracle.cnmf_oracle.dense_lowrank), fp32-rounded."""
    g = np.random.default_rng(seed)
    x = g.uniform(size=(m, 20))
    y = g.uniform(size=(20, n))
    a = np.maximum(x @ y + 0.01 * g.standard_normal((m, n)), 0.0)
    return a.astype(np.float32).astype(np.float64)


def perturbed(a, k):
    xi = np.random.default_rng(5000 + k).standard_normal(a.shape)
    return a * (1.0 + 2.0 ** -24 * xi)


def proj_dist(q1, q2):
    return float(np.linalg.norm(q2 - q1 @ (q1.T @ q2), 2))


def main():
    sys.path.insert(0, REF)
    import cnmf
    from cnmf import CompressionConfig

    from oracle import cnmf_oracle as O

    fx = {}
    for (m, n) in ((2000, 1000), (10000, 5000)):
        a = dense_config1(m, n, seed=11)
        cfg = CompressionConfig(r=20, r_ov=10, w=4, seed=3)
        q = cnmf.structured_compress(a, cfg, reorthogonalize=True).q_dense()
        band = [proj_dist(q, cnmf.structured_compress(perturbed(a, k), cfg, reorthogonalize=True).q_dense())
                for k in range(3)]
        q_stock = cnmf.structured_compress(a, cfg).q_dense()
        key = f"c1_{m}x{n}"
        fx[key + "_q"] = q.astype(np.float32)
        fx[key + "_band"] = np.array(band)
        fx[key + "_stock_dist"] = np.float64(proj_dist(q, q_stock))
        fx[key + "_err_reorth"] = np.float64(cnmf.compression_error(a, cnmf.structured_compress(
            a, cfg, reorthogonalize=True)))
        fx[key + "_err_stock"] = np.float64(cnmf.compression_error(a, cnmf.structured_compress(a, cfg)))
        print(key, "band", band, "stock distance", fx[key + "_stock_dist"], flush=True)

    for seed in (1, 2):
        a, truth = O.near_separable(2_000_000, 200, 20, 0.5, 0.005, seed=seed)
        a = a.astype(np.float32).astype(np.float64)
        outcomes, picks0 = [], None
        for k in range(4):
            ak = a if k == 0 else perturbed(a, 100 + k)
            cfg = cnmf.adjust_config(CompressionConfig(r=20, r_ov=10, w=2, seed=7), *ak.shape)
            q = cnmf.structured_compress(ak, cfg, reorthogonalize=True).q_dense()
            red = q.T @ ak
            picks = np.asarray(cnmf.select_columns_spa(red, 20))
            if k == 0:
                picks0 = picks
            assert np.array_equal(picks, picks0), "picks moved under a 2^-24 perturbation"
            try:
                cnmf.snmf_right_factor(red, picks)
                outcomes.append(1)  # returns
            except cnmf.ConvergenceError:
                outcomes.append(0)  # exchange cap
            print("configs[2] seed", seed, "perturbation", k, "returns" if outcomes[-1] else "raises", flush=True)
        fx[f"c2_seed{seed}_picks"] = picks0
        fx[f"c2_seed{seed}_truth"] = np.asarray(truth)
        fx[f"c2_seed{seed}_nnls_returns"] = np.array(outcomes)
    np.savez_compressed(OUT, **fx)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
