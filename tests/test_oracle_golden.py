"""Pin the CPU oracle to the reference: every oracle function reproduces the
fixtures written by running the reference package (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import cnmf_oracle as O


def test_child_seeds(golden):
    tags = list(golden["child_seed_tags"])
    got = [O.child_seed(int(s), tags[int(i)]) for s, i in golden["child_seed_in"]]
    assert np.array_equal(np.array(got, dtype=np.uint64), golden["child_seed_out"])


def test_test_matrix_bitexact(golden):
    assert np.array_equal(O.test_matrix(4100, 3, 3), golden["omega_4100x3_seed3"])
    assert np.array_equal(O.test_matrix(300, 30, 99), golden["omega_300x30_seed99"])
    assert np.array_equal(O.generator(42).standard_normal((10, 7)), golden["gauss_10x7_seed42"])


def test_uniform_init_bitexact(golden):
    assert np.array_equal(O.uniform_matrix(5, "init-left", (30, 4)), golden["uniform_init_left_seed5"])


def test_adjust(golden):
    got = [(c.r, c.r_ov) for c in (O.adjust(O.Config(5, 10), 2000, 1000),
                                   O.adjust(O.Config(5, 10), 2000, 12),
                                   O.adjust(O.Config(30, 10), 2000, 1000))]
    assert np.array_equal(np.array(got), golden["adjust"])
    with pytest.raises(O.OracleError):
        O.adjust(O.Config(12), 50, 12)


@pytest.mark.parametrize("w", [0, 2])
def test_range_basis(golden, w):
    a = golden["cmp_a"]
    cfg = O.Config(r=8, r_ov=12, w=w, seed=3)
    assert np.abs(O.range_basis(a, cfg, reorth=False) - golden[f"cmp_q_w{w}"]).max() < 1e-12
    assert np.abs(O.range_basis(a, cfg, reorth=True) - golden[f"cmp_q_w{w}_reorth"]).max() < 1e-12
    assert np.abs(O.row_basis(a, cfg, reorth=True) - golden[f"cmp_qrows_w{w}_reorth"]).max() < 1e-12


def test_reorth_flag_same_subspace(golden):
    # both reference settings define the same Q (well-conditioned input)
    assert np.abs(golden["cmp_q_w2"] - golden["cmp_q_w2_reorth"]).max() < 1e-6
    q = O.range_basis(golden["cmp_a"], O.Config(r=8, r_ov=12, w=2, seed=3), reorth=False)
    assert abs(O.residual_norm(golden["cmp_a"], q) - float(golden["cmp_err_w2"])) < 1e-9


def test_nnls(golden):
    assert np.abs(O.nnls(golden["nnls_c"], golden["nnls_d"]) - golden["nnls_h"]).max() < 1e-12


def test_selectors(golden):
    a = golden["sep_a"]
    assert np.array_equal(O.spa(a, 6), golden["spa_picks"])
    assert np.array_equal(O.xray(a, 6), golden["xray_picks"])
    assert np.array_equal(O.spa(golden["spa_noisy_in"], 6), golden["spa_noisy_picks"])
    assert set(golden["spa_picks"].tolist()) == set(golden["sep_truth"].tolist())


@pytest.mark.parametrize("sel", ["spa", "xray"])
def test_snmf_pipeline(golden, sel):
    out = O.snmf(golden["sep_a"], 6, selector=sel, cfg=O.Config(r=6, r_ov=10, w=2, seed=9), reorth=False)
    assert np.array_equal(out.K, golden[f"snmf_{sel}_K"])
    assert np.abs(out.Y - golden[f"snmf_{sel}_Y"]).max() < 1e-9
    assert np.allclose([out.rel_error_reduced, out.rel_error_full], golden[f"snmf_{sel}_err"], atol=1e-12)


def test_admm_identity_path(golden):
    seen = []
    O.admm(golden["admm_a"], 3, compressed=False, cfg=O.Config(r=3, seed=7), max_iter=12, tol=0.0,
           on_iteration=lambda k, st: seen.append(np.concatenate([x.ravel() for x in st])))
    assert np.abs(np.array(seen) - golden["admm_plain_states"]).max() < 1e-10


def test_admm_compressed(golden):
    bases = (golden["admm_comp_left"], golden["admm_comp_right"])
    out = O.admm(golden["admm_a"], 3, compressed=True, cfg=O.Config(r=3, seed=7), max_iter=300,
                 tol=1e-6, bases=bases)
    it, rel = golden["admm_comp_meta"]
    assert out.iterations == int(it)
    assert abs(out.rel_error - rel) < 1e-10
    assert np.abs(np.array(out.trace) - golden["admm_comp_trace"]).max() < 1e-9
    assert np.abs(out.X - golden["admm_comp_X"]).max() < 1e-9
    # the reference bases are reproduced by the oracle's reorth=False path
    cfg = O.adjust(O.Config(r=3, seed=7), 40, 30)
    left, right = O.compressed_bases(golden["admm_a"], cfg, reorth=False)
    assert np.abs(left - bases[0]).max() < 1e-12 and np.abs(right - bases[1]).max() < 1e-12


def test_kkt(golden):
    left, right = golden["admm_comp_left"], golden["admm_comp_right"]
    s, r, m, n = left.shape[1], 3, 40, 30
    st = golden["kkt_state5"]
    sizes = [s * r, r * s, m * r, r * n, m * r, r * n]
    shapes = [(s, r), (r, s), (m, r), (r, n), (m, r), (r, n)]
    parts, off = [], 0
    for sz, sh in zip(sizes, shapes):
        parts.append(st[off:off + sz].reshape(sh))
        off += sz
    core = left.T @ golden["admm_a"] @ right.T
    assert np.allclose(O.kkt(*parts, core, left, right), golden["kkt_vals5"], rtol=1e-12, atol=1e-14)


def test_rel_error(golden):
    assert abs(O.rel_error(golden["admm_a"], golden["admm_comp_X"], golden["admm_comp_Y"])
               - golden["relerr"][0]) < 1e-14
