"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py

It imports ``cnmf`` from /root/reference/pkg/src, runs it on small seeded
inputs and writes ``tests/golden/reference_vectors.npz``. The fixture is
committed; neither the tests nor the GPU box ever read /root/reference.
"""

import os
import sys
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.npz")


def main():
    sys.path.insert(0, REF)
    import cnmf
    from cnmf import CompressionConfig, Rng
    from cnmf.compress import draw_test_matrix

    fx = {}
    # --- RNG: child seeds, test matrix (two 4096-row chunks), uniform init ---
    tags = ["omega", "chunk0", "chunk1", "left-basis", "right-basis", "init-left", "init-right", "é-ü"]
    seeds = [0, 1, 7, 12345, 2**63 + 11, 2**64 - 1]
    fx["child_seed_in"] = np.array([[s, i] for s in seeds for i in range(len(tags))], dtype=np.uint64)
    fx["child_seed_out"] = np.array([cnmf.child_seed(s, t) for s in seeds for t in tags], dtype=np.uint64)
    fx["child_seed_tags"] = np.array(tags)
    fx["omega_4100x3_seed3"] = draw_test_matrix(CompressionConfig(r=2, r_ov=1, w=0, seed=3), 4100)
    fx["omega_300x30_seed99"] = draw_test_matrix(CompressionConfig(r=20, r_ov=10, w=0, seed=99), 300)
    fx["gauss_10x7_seed42"] = cnmf.gaussian_matrix(10, 7, Rng(42))
    fx["uniform_init_left_seed5"] = Rng(5).child("init-left").uniform((30, 4))

    # --- structured compression (reference default and reorthogonalized) ---
    g = np.random.default_rng(1)
    a = g.standard_normal((120, 90)) @ np.diag(0.9 ** np.arange(90)) @ g.standard_normal((90, 90))
    fx["cmp_a"] = a
    for w in (0, 2):
        cfg = CompressionConfig(r=8, r_ov=12, w=w, seed=3)
        fx[f"cmp_q_w{w}"] = cnmf.structured_compress(a, cfg).q_dense()
        fx[f"cmp_q_w{w}_reorth"] = cnmf.structured_compress(a, cfg, reorthogonalize=True).q_dense()
        fx[f"cmp_qrows_w{w}_reorth"] = cnmf.structured_compress_rows(a, cfg, reorthogonalize=True).q_dense()
    fx["cmp_err_w2"] = np.float64(cnmf.compression_error(a, cnmf.structured_compress(
        a, CompressionConfig(r=8, r_ov=12, w=2, seed=3))))
    fx["adjust"] = np.array([
        [c.r, c.r_ov] for c in (
            cnmf.adjust_config(CompressionConfig(r=5, r_ov=10), 2000, 1000),
            cnmf.adjust_config(CompressionConfig(r=5, r_ov=10), 2000, 12),
            cnmf.adjust_config(CompressionConfig(r=30, r_ov=10), 2000, 1000))])

    # --- NNLS ---
    c = g.standard_normal((25, 10))
    d = g.standard_normal((25, 6))
    fx["nnls_c"], fx["nnls_d"] = c, d
    fx["nnls_h"] = cnmf.nnls_solve(c, d)

    # --- SPA / XRAY / snmf on a small near-separable instance ---
    store, truth = cnmf.gen_separable_synthetic(60, 300, 6, noise=0.0, seed=4)
    sep = store.to_dense()
    fx["sep_a"], fx["sep_truth"] = sep, truth
    fx["spa_picks"] = cnmf.select_columns_spa(sep, 6)
    fx["xray_picks"] = cnmf.select_columns_xray(sep, 6)
    cfg = CompressionConfig(r=6, r_ov=10, w=2, seed=9)
    for sel in ("spa", "xray"):
        res = cnmf.snmf(sep, 6, selector=sel, reduction="compressed", cfg=cfg)
        fx[f"snmf_{sel}_K"] = res.K
        fx[f"snmf_{sel}_Y"] = res.Y
        fx[f"snmf_{sel}_err"] = np.array([res.rel_error_reduced, res.rel_error_full])
    # SPA on noisy data (not exactly separable)
    fx["spa_noisy_in"] = sep + 0.01 * g.standard_normal(sep.shape)
    fx["spa_noisy_picks"] = cnmf.select_columns_spa(fx["spa_noisy_in"], 6)

    # --- ADMM: identity path iterates, compressed run trace, KKT ---
    x = Rng(5).child("x").uniform((40, 3))
    y = Rng(5).child("y").uniform((3, 30))
    an = x @ y + 0.05 * Rng(6).standard_normal((40, 30))
    fx["admm_a"] = an
    seen = []
    cnmf.nmf_admm(an, 3, compressed=False, cfg=CompressionConfig(r=3, seed=7), max_iter=12, tol=0.0,
                  on_iteration=lambda k, st: seen.append(np.concatenate(
                      [st.xc.ravel(), st.yc.ravel(), st.u.ravel(), st.v.ravel(),
                       st.dual_u.ravel(), st.dual_v.ravel()])))
    fx["admm_plain_states"] = np.array(seen)
    states = []
    fp = cnmf.nmf_admm(an, 3, compressed=True, cfg=CompressionConfig(r=3, seed=7), max_iter=300,
                       tol=1e-6, on_iteration=lambda k, st: states.append(st))
    fx["admm_comp_trace"] = np.array(fp.objective_trace)
    fx["admm_comp_X"], fx["admm_comp_Y"] = fp.X, fp.Y
    fx["admm_comp_meta"] = np.array([fp.iterations, fp.rel_error])
    cfg = cnmf.adjust_config(CompressionConfig(r=3, seed=7), 40, 30)
    left = cnmf.structured_compress(an, replace(cfg, seed=cnmf.child_seed(7, "left-basis"))).q_dense()
    right = cnmf.structured_compress_rows(
        an, replace(cfg, seed=cnmf.child_seed(7, "right-basis"))).q_dense().T
    fx["admm_comp_left"], fx["admm_comp_right"] = left, right
    st = states[5]
    core = left.T @ an @ right.T
    k = cnmf.kkt_residual(st, core, left, right)
    fx["kkt_state5"] = np.concatenate([st.xc.ravel(), st.yc.ravel(), st.u.ravel(), st.v.ravel(),
                                       st.dual_u.ravel(), st.dual_v.ravel()])
    fx["kkt_vals5"] = np.array([k.grad_left, k.grad_right, k.feas_left, k.feas_right,
                                k.comp_left, k.comp_right])
    fx["relerr"] = np.array([cnmf.relative_error(an, fp.X, fp.Y)])

    np.savez_compressed(OUT, **fx)
    print("wrote", OUT, sum(np.asarray(v).nbytes for v in fx.values()), "bytes")


if __name__ == "__main__":
    main()
