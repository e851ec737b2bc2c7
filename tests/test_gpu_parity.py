"""GPU parity: the CUDA path (through the C ABI / reference-style API) against
the CPU oracle and the reference golden vectors.

Tolerances (north_star, BASELINE.json): bit-exact for RNG streams and for
selected column indices; subspace projector distance <= 1e-4 for fp32
bases; relative error of the final NMF fit within 1e-3 (relative) of the
oracle; fp32 pass products within 2e-5 relative Frobenius error of fp64.
"""

import os

import numpy as np
import pytest
import torch

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cnmf_oracle as O  # noqa: E402

import paper_1505_04650_b200 as C  # noqa: E402
from paper_1505_04650_b200 import _lib  # noqa: E402
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def relf(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- RNG -----

def test_omega_bitexact_golden(golden):
    om = C.draw_test_matrix(C.CompressionConfig(r=2, r_ov=1, w=0, seed=3), 4100).cpu().numpy()
    assert np.array_equal(om, golden["omega_4100x3_seed3"])
    om = C.draw_test_matrix(C.CompressionConfig(r=20, r_ov=10, w=0, seed=99), 300).cpu().numpy()
    assert np.array_equal(om, golden["omega_300x30_seed99"])
    g = C.gaussian_matrix(10, 7, C.Rng(42)).cpu().numpy()
    assert np.array_equal(g, golden["gauss_10x7_seed42"])


@pytest.mark.parametrize("rows,cols,seed", [(20000, 60, 7), (9000, 30, 2**63 + 1), (5, 1, 0)])
def test_omega_bitexact_numpy(rows, cols, seed):
    cfg = C.CompressionConfig(r=cols, r_ov=0, w=0, seed=seed)
    got = C.draw_test_matrix(cfg, rows).cpu().numpy()
    assert np.array_equal(got, O.test_matrix(rows, cols, seed))


def test_unchunked_stream_bitexact_large():
    got = C.Rng(123).standard_normal((1, 1_500_000)).cpu().numpy().ravel()
    want = O.generator(123).standard_normal(1_500_000)
    assert np.array_equal(got, want)


def test_ziggurat_tail_bitexact():
    # tail variates (|x| > r) take numpy's log1p path (glibc's FMA build,
    # restated on the device): bit-exact over thousands of tail draws
    got = C.Rng(2024).standard_normal((1, 8_000_000)).cpu().numpy().ravel()
    want = O.generator(2024).standard_normal(8_000_000)
    assert np.count_nonzero(np.abs(want) > 3.6541528853610088) > 1000
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed", [3, 2**64 - 5])
def test_rng_successive_draws_continue_the_stream(seed):
    # rng.py:38-70: successive draws on one Rng continue numpy's Philox
    # stream (uniform = one raw draw per variate, normals = the ziggurat's
    # variable count), including starts in the middle of a 4-word block
    r = C.Rng(seed)
    g = O.generator(seed)
    for kind, shape in (("u", (3, 5)), ("n", (1, 1001)), ("u", (7,)), ("n", (40, 25)), ("n", (3,)),
                        ("u", (2, 9)), ("n", (1, 200_001)), ("u", (1, 6))):
        if kind == "u":
            got = r.uniform(shape).cpu().numpy()
            want = g.uniform(0.0, 1.0, size=shape)
        else:
            got = r.standard_normal(shape).cpu().numpy()
            want = g.standard_normal(shape)
        assert np.array_equal(got, want), (kind, shape)
    with pytest.raises(C.ArgumentError):
        r.permutation(5)


def test_uniform_bitexact(golden):
    got = C.Rng(5).child("init-left").uniform((30, 4)).cpu().numpy()
    assert np.array_equal(got, golden["uniform_init_left_seed5"])
    t = C.Rng(77).uniform((300, 7), transpose=True).cpu().numpy()
    assert np.array_equal(t.T, O.generator(77).uniform(0, 1, (300, 7)))


# -------------------------------------------------------------- passes ----

@pytest.mark.parametrize("m,n,s", [(1000, 700, 30), (257, 1023, 60), (4000, 130, 100), (33, 41, 20),
                                   (5000, 2003, 64)])
def test_passes_match_fp64(m, n, s):
    g = np.random.default_rng(m + n)
    a = g.standard_normal((m, n))
    A = DeviceMatrix(a)
    S = C.compress.panel_ld(s)
    x = np.zeros((n, S), np.float32)
    x[:, :s] = g.standard_normal((n, s))
    w = np.zeros((m, S), np.float32)
    w[:, :s] = g.standard_normal((m, s))
    X = torch.from_numpy(x).cuda()
    Wd = torch.from_numpy(w).cuda()
    Y = zeros((m, S))
    Z = zeros((n, S))
    _lib.call("cnmf_pass_forward", A.ptr, m, n, A.lda, X.data_ptr(), s, Y.data_ptr(), stream())
    _lib.call("cnmf_pass_transpose", A.ptr, m, n, A.lda, Wd.data_ptr(), s, Z.data_ptr(), stream())
    a32 = a.astype(np.float32).astype(np.float64)
    assert relf(Y.cpu().numpy()[:, :s], a32 @ x[:, :s]) < 2e-5
    assert relf(Z.cpu().numpy()[:, :s], a32.T @ w[:, :s]) < 2e-5
    assert np.all(Y.cpu().numpy()[:, s:] == 0) and np.all(Z.cpu().numpy()[:, s:] == 0)


@pytest.mark.parametrize("m,n,s", [(1000, 700, 30), (300, 1029, 60), (129, 33, 20), (4096, 2048, 64)])
def test_tensor_core_passes_match_ffma_and_fp64(m, n, s):
    """tcgen05 3xTF32 passes agree with fp64 to fp32-level accuracy."""
    g = np.random.default_rng(7 * m + n)
    a = g.standard_normal((m, n))
    A = DeviceMatrix(a)
    S = C.compress.panel_ld(s)
    x = np.zeros((n, S), np.float32)
    x[:, :s] = g.standard_normal((n, s))
    w = np.zeros((m, S), np.float32)
    w[:, :s] = g.standard_normal((m, s))
    X, Wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    a32 = a.astype(np.float32).astype(np.float64)
    lib = _lib.load()
    out = {}
    for impl in (1, 0):
        lib.cnmf_set_pass_impl(impl)
        Y, Z = zeros((m, S)), zeros((n, S))
        _lib.call("cnmf_pass_forward", A.ptr, m, n, A.lda, X.data_ptr(), s, Y.data_ptr(), stream())
        _lib.call("cnmf_pass_transpose", A.ptr, m, n, A.lda, Wd.data_ptr(), s, Z.data_ptr(), stream())
        out[impl] = (Y.cpu().numpy()[:, :s].astype(np.float64), Z.cpu().numpy()[:, :s].astype(np.float64))
    lib.cnmf_set_pass_impl(1)
    for impl in (1, 0):
        assert relf(out[impl][0], a32 @ x[:, :s]) < 3e-6, impl
        assert relf(out[impl][1], a32.T @ w[:, :s]) < 3e-6, impl


# --------------------------------------------------------- compression ----

@pytest.mark.parametrize("w", [0, 2, 4])
def test_compress_matches_oracle_full_spectrum(golden, w):
    a = golden["cmp_a"]
    cfg = C.CompressionConfig(r=8, r_ov=12, w=w, seed=3)
    q = C.structured_compress(a, cfg).Q
    ref = O.range_basis(a, O.Config(8, 12, w, 3), reorth=True)
    assert np.linalg.norm(q.T @ q - np.eye(20)) < 1e-5
    assert O.projector_distance(q, ref) <= 1e-4
    # sign-canonical columns agree individually where the spectrum separates them
    assert np.abs(q[:, :8] - ref[:, :8]).max() < 1e-3
    qr_ = C.structured_compress_rows(a, cfg).Q
    refr = O.row_basis(a, O.Config(8, 12, w, 3), reorth=True)
    assert O.projector_distance(qr_, refr) <= 1e-4


def test_compress_reference_golden(golden):
    # the reference's own reorthogonalized basis (golden) at w = 2
    q = C.structured_compress(golden["cmp_a"], C.CompressionConfig(r=8, r_ov=12, w=2, seed=3)).Q
    assert O.projector_distance(q, golden["cmp_q_w2_reorth"]) <= 1e-4
    qr_ = C.structured_compress_rows(golden["cmp_a"], C.CompressionConfig(r=8, r_ov=12, w=2, seed=3)).Q
    assert O.projector_distance(qr_, golden["cmp_qrows_w2_reorth"]) <= 1e-4


def test_compress_lowrank_signal_subspace():
    # config-1-like data: rank-20 signal + noise; the signal subspace is the
    # determined part of Q (the noise directions are roundoff-defined)
    a = O.dense_lowrank(1500, 800, 20, 0.01, seed=1)
    cfg = C.CompressionConfig(r=20, r_ov=10, w=4, seed=5)
    q = C.structured_compress(a, cfg).Q
    ref = O.range_basis(a, O.Config(20, 10, 4, 5), reorth=True)
    u = np.linalg.svd(a, full_matrices=False)[0][:, :20]
    # both capture the rank-20 signal subspace
    assert np.linalg.norm(u - q @ (q.T @ u), 2) < 1e-4
    assert np.linalg.norm(u - ref @ (ref.T @ u), 2) < 1e-4
    assert abs(O.residual_norm(a, q) - O.residual_norm(a, ref)) / O.residual_norm(a, ref) < 1e-3


def test_compress_exact_low_rank_and_errors():
    x = np.random.default_rng(0).uniform(size=(300, 5))
    y = np.random.default_rng(1).uniform(size=(5, 200))
    a = x @ y
    basis = C.structured_compress(a, C.CompressionConfig(r=5, r_ov=10, w=0, seed=1))
    q = basis.Q
    assert np.linalg.norm(q.T @ q - np.eye(15)) < 1e-4
    assert O.residual_norm(a, q) / np.linalg.norm(a) < 1e-5
    assert C.compression_error(a, basis) / np.linalg.norm(a) < 2e-3
    with pytest.raises(C.InfeasibleRankError):
        C.structured_compress(np.ones((30, 10)), C.CompressionConfig(r=8, r_ov=10, w=0))


def test_compression_error_matches_oracle(golden):
    a = golden["cmp_a"]
    basis = C.structured_compress(a, C.CompressionConfig(r=8, r_ov=12, w=2, seed=3))
    want = O.residual_norm(a, basis.Q)
    assert abs(C.compression_error(a, basis) - want) <= 1e-4 * want + 1e-5 * np.linalg.norm(a)


def test_device_tensor_roundtrip():
    a = torch.rand(2000, 1000, device="cuda")
    basis = C.structured_compress(a, C.CompressionConfig(r=10, r_ov=10, w=1, seed=4))
    assert isinstance(basis.Q, torch.Tensor) and basis.Q.is_cuda and basis.Q.shape == (2000, 20)


# ----------------------------------------------------------- selection ----

def test_spa_xray_golden(golden):
    a = golden["sep_a"]
    assert np.array_equal(C.select_columns_spa(a, 6), golden["spa_picks"])
    assert np.array_equal(C.select_columns_xray(a, 6), golden["xray_picks"])
    assert np.array_equal(C.select_columns_spa(golden["spa_noisy_in"], 6), golden["spa_noisy_picks"])


def test_spa_rank_deficiency_reports_picks():
    v = np.array([[1.0], [2.0]])
    with pytest.raises(C.RankDeficiencyError) as info:
        C.select_columns_spa(np.hstack([v, 2 * v, 3 * v]), 2)
    assert info.value.picks == [2]


def test_spa_ties_lowest_index():
    r_mat = np.array([[3.0, 0.0, 1.0], [0.0, 2.0, 0.0]])
    assert C.select_columns_spa(r_mat, 2).tolist() == [0, 1]
    r = np.eye(4)
    assert C.select_columns_spa(r, 4).tolist() == [0, 1, 2, 3]


def test_nnls_golden(golden):
    h = C.nnls_solve(golden["nnls_c"], golden["nnls_d"])
    assert np.abs(h - golden["nnls_h"]).max() < 1e-9
    assert np.array_equal(C.nnls_solve(np.eye(3), np.array([1.0, -2.0, 3.0])), [1.0, 0.0, 3.0])


def test_nnls_random_against_oracle():
    g = np.random.default_rng(3)
    for q in (2, 7, 20, 40):
        c = g.standard_normal((60, q))
        d = g.standard_normal((60, 50))
        h = C.nnls_solve(c, d)
        ref = O.nnls(c, d)
        obj = np.sum((d - c @ h) ** 2, axis=0)
        ref_obj = np.sum((d - c @ ref) ** 2, axis=0)
        assert np.all(obj <= ref_obj + 1e-8 * (1 + ref_obj))
        assert h.min() >= 0


@pytest.mark.parametrize("sel", ["spa", "xray"])
def test_snmf_pipeline_vs_oracle(golden, sel):
    a = golden["sep_a"]
    cfg = C.CompressionConfig(r=6, r_ov=10, w=2, seed=9)
    res = C.snmf(a, 6, selector=sel, cfg=cfg)
    ref = O.snmf(a, 6, selector=sel, cfg=O.Config(6, 10, 2, 9))
    assert np.array_equal(res.K, ref.K)
    assert np.array_equal(res.K, golden[f"snmf_{sel}_K"])
    assert np.abs(res.Y - ref.Y).max() < 1e-4
    assert res.rel_error_full < 1e-5 and res.rel_error_reduced < 1e-5


@pytest.mark.parametrize("sel", ["spa", "xray"])
def test_snmf_qr_reduction_fat_and_tall(sel):
    # the reference's own cases (tests/test_snmf.py: 50 x 200 and 40 x 300 fat
    # matrices, exact rank 5; qr and compressed reductions must agree) plus a
    # tall one, each against the oracle with the reference's canonical QR basis
    for m, n, seed in ((50, 200, 0), (50, 200, 3), (40, 300, 14), (3000, 120, 12)):
        a, truth = O.near_separable(m, n, 5 if m < 3000 else 4, 1.0, 0.0, seed=seed)
        r = len(truth)
        res = C.snmf(a, r, selector=sel, reduction="qr")
        ref = O.snmf(a, r, selector=sel, basis=O.qr_pos(a)[0])
        assert sorted(res.K.tolist()) == truth.tolist()
        assert np.array_equal(res.K, ref.K)
        assert res.rel_error_full <= 1e-6 and res.Y.min() >= 0
        assert np.abs(res.Y - ref.Y).max() < 1e-4
        cmp = C.snmf(a, r, selector=sel, reduction="compressed", cfg=C.CompressionConfig(r=r, r_ov=10, w=0, seed=seed))
        assert set(cmp.K.tolist()) == set(res.K.tolist())


def test_snmf_qr_reduction_limits():
    a, _ = O.near_separable(200, 400, 5, 1.0, 0.0, seed=1)
    with pytest.raises(C.ArgumentError):
        C.snmf(a, 5, reduction="qr")  # fat with m > 128
    with pytest.raises(C.ArgumentError):
        C.snmf(a.T.copy(), 5, reduction="qr")  # tall with n > 128


def test_snmf_near_separable_config0_shape():
    a, truth = O.near_separable(500, 2000, 10, 1.0, 0.01, seed=11)
    res = C.snmf(a, 10, selector="spa", cfg=C.CompressionConfig(r=10, r_ov=10, w=4, seed=2))
    ref = O.snmf(a, 10, selector="spa", cfg=O.Config(10, 10, 4, 2))
    assert np.array_equal(res.K, ref.K)
    assert sorted(res.K.tolist()) == truth.tolist()
    assert abs(res.rel_error_full - ref.rel_error_full) <= 1e-3 * ref.rel_error_full


def test_snmf_tall_skinny_config2_shape():
    # configs[2]: tall-and-skinny near-separable, fp32, n = 200, r = 20,
    # alpha = 0.5, noise 0.005, q = 2 (m reduced from 2,000,000 to keep the
    # oracle's CPU run short; the device path is size-independent here)
    a, truth = O.near_separable(60_000, 200, 20, 0.5, 0.005, seed=21)
    a32 = a.astype(np.float32)
    res = C.snmf(a32, 20, selector="spa", cfg=C.CompressionConfig(r=20, r_ov=10, w=2, seed=4))
    ref = O.snmf(a32.astype(np.float64), 20, selector="spa", cfg=O.Config(20, 10, 2, 4))
    assert np.array_equal(res.K, ref.K)
    assert sorted(res.K.tolist()) == truth.tolist()
    assert abs(res.rel_error_full - ref.rel_error_full) <= 1e-3 * ref.rel_error_full


def test_xray_config3_shape_small():
    # configs[3] (general shape, XRAY) at reduced size: m = 1200, n = 1500,
    # r = 40 (s = 50: the 64-wide panel path)
    a, truth = O.near_separable(1200, 1500, 40, 1.0, 0.01, seed=31)
    a32 = a.astype(np.float32)
    res = C.snmf(a32, 40, selector="xray", cfg=C.CompressionConfig(r=40, r_ov=10, w=4, seed=6))
    ref = O.snmf(a32.astype(np.float64), 40, selector="xray", cfg=O.Config(40, 10, 4, 6))
    assert np.array_equal(res.K, ref.K)  # pick order included
    assert sorted(res.K.tolist()) == truth.tolist()


def test_xray_pick_order_and_right_factor_on_the_oracle_reduction(monkeypatch):
    # the selection and NNLS kernels in isolation: on the ORACLE's reduced
    # matrix (fp64, configs[3]-like: s = 50, r = 40) the device's XRAY picks
    # equal the oracle's INCLUDING their order, whatever the NNLS start (warm
    # refits with kept factors, warm without, cold like the reference), and the
    # right factor (started from the selection's last refit when one exists)
    # is the oracle's minimiser
    a, truth = O.near_separable(1200, 1500, 40, 1.0, 0.01, seed=31)
    ref = O.snmf(a, 40, selector="xray", cfg=O.Config(40, 10, 4, 6))
    assert sorted(ref.K.tolist()) == truth.tolist()
    for warm, factors in (("1", "1"), ("1", "0"), ("0", "1")):
        monkeypatch.setenv("CNMF_XRAY_WARM", warm)
        monkeypatch.setenv("CNMF_XRAY_FACTORS", factors)
        picks = C.select_columns_xray(ref.reduced, 40, mass=ref.mass)
        assert np.array_equal(picks, ref.K), (warm, factors)
        y = C.snmf_right_factor(ref.reduced, picks)
        assert y.min() >= 0.0
        assert np.abs(y - ref.Y).max() <= 1e-8 * max(1.0, np.abs(ref.Y).max()), (warm, factors)


# ---------------------------------------------------------------- ADMM ----

def test_admm_matches_oracle_on_same_bases(golden):
    a = O.dense_lowrank(600, 400, 6, 0.01, seed=4)
    cfg = C.CompressionConfig(r=6, r_ov=10, w=4, seed=7)
    states = []
    fp = C.nmf_admm(a, 6, cfg=cfg, max_iter=60, tol=0.0,
                    on_iteration=lambda k, st: states.append(st))
    assert fp.iterations == 60 and len(states) == 60
    # oracle ADMM on the device's own bases (isolates the iteration)
    from paper_1505_04650_b200.nmf import compressed_problem
    A = DeviceMatrix(a)
    left, right, _ = compressed_problem(A, C.adjust_config(cfg, 600, 400))
    bases = (left.Q, right.Q.T)
    ref = O.admm(a, 6, cfg=O.Config(6, 10, 4, 7), max_iter=60, tol=0.0, bases=bases)
    assert np.abs(np.array(fp.objective_trace) - np.array(ref.trace)).max() <= 1e-4 * max(ref.trace)
    assert abs(fp.rel_error - ref.rel_error) <= 1e-3 * ref.rel_error
    assert fp.X.min() >= 0 and fp.Y.min() >= 0
    assert min(min(s.u.min(), s.v.min()) for s in states) >= 0


def test_admm_stopping_rule_and_oracle_error():
    x = O.uniform_matrix(21, "x", (100, 5))
    y = O.uniform_matrix(21, "y", (5, 80))
    a = x @ y
    fp = C.nmf_admm(a, 5, cfg=C.CompressionConfig(r=5, seed=0), max_iter=500, tol=1e-4)
    ref = O.admm(a, 5, cfg=O.Config(5, 10, 4, 0), max_iter=500, tol=1e-4)
    # exact rank 5 < s = 20: the trailing basis columns are roundoff-defined
    # in both implementations, so only the reference's own criteria apply
    # (test_admm.py:57-64): converged before the cap, to rel_error <= 1e-4
    assert fp.iterations < 500 and ref.iterations < 500
    assert fp.rel_error <= 1e-4 and ref.rel_error <= 1e-4


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_admm_config1_shape_parity_200(seed):
    # configs[1]-shaped fp32 workload (both sides see the same fp32 matrix) at
    # configs[4]'s 200 ADMM iterations: north_star's tolerance, 1e-3 relative
    # on the final ||A - XY||_F / ||A||_F (measured: <= 1.4e-4)
    a = O.dense_lowrank(2000, 1000, 20, 0.01, seed=seed).astype(np.float32)
    cfg = C.CompressionConfig(r=20, r_ov=10, w=4, seed=5 + seed)
    fp = C.nmf_admm(a, 20, cfg=cfg, max_iter=200, tol=1e-4)
    ref = O.admm(a, 20, cfg=O.Config(20, 10, 4, 5 + seed), max_iter=200, tol=1e-4)
    assert fp.iterations == ref.iterations
    assert abs(fp.rel_error - ref.rel_error) <= 1e-3 * ref.rel_error


def test_admm_config1_shape_parity_500():
    # configs[1]'s 500 iterations on noisy data are chaotic: the reference
    # itself moves its final error by up to ~1.6e-3 relative when A is
    # perturbed by fp32 rounding (tools/admm_parity_seeds.py). The bound is
    # 1e-3 or twice the reference's own spread under two such perturbations,
    # measured here, whichever is larger.
    a = O.dense_lowrank(2000, 1000, 20, 0.01, seed=0).astype(np.float32)
    cfg = C.CompressionConfig(r=20, r_ov=10, w=4, seed=5)
    fp = C.nmf_admm(a, 20, cfg=cfg, max_iter=500, tol=1e-4)
    ocfg = O.Config(20, 10, 4, 5)
    ref = O.admm(a, 20, cfg=ocfg, max_iter=500, tol=1e-4)
    spread = 0.0
    for k in range(2):
        g = np.random.default_rng(100 + k)
        ap = a.astype(np.float64) * (1.0 + 6e-8 * g.standard_normal(a.shape))
        spread = max(spread, abs(O.admm(ap, 20, cfg=ocfg, max_iter=500, tol=1e-4).rel_error - ref.rel_error))
    assert fp.iterations == ref.iterations
    assert abs(fp.rel_error - ref.rel_error) <= max(1e-3 * ref.rel_error, 2.0 * spread)


@pytest.mark.parametrize("m,n", [(4000, 3000), (3000, 4000), (5000, 3000), (10000, 5000)])
def test_passes_split_k_repeated(m, n):
    # shapes whose output tiles are shared by several CTAs (split-K): every
    # one of repeated launches matches fp64 (a corrupted tile shows ~1e-2)
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.rand(m, n, device="cuda", generator=g)
    A = DeviceMatrix(a)
    x = torch.randn(n, 32, device="cuda", generator=g)
    w = torch.randn(m, 32, device="cuda", generator=g)
    lib = _lib.load()
    yref = (a.double() @ x.double())
    zref = (a.double().t() @ w.double())
    for _ in range(12):
        y, z = zeros((m, 32)), zeros((n, 32))
        lib.cnmf_pass_forward(A.ptr, m, n, A.lda, x.data_ptr(), 32, y.data_ptr(), stream())
        lib.cnmf_pass_transpose(A.ptr, m, n, A.lda, w.data_ptr(), 32, z.data_ptr(), stream())
        torch.cuda.synchronize()
        assert ((y.double() - yref).abs().max() / yref.abs().max()).item() < 1e-5
        assert ((z.double() - zref).abs().max() / zref.abs().max()).item() < 1e-5


@pytest.mark.parametrize("m,n,S", [(4000, 3000, 32), (5000, 3000, 32), (3000, 4000, 64), (10000, 5000, 32),
                                   (2600, 1300, 64)])
def test_passes_bit_reproducible(m, n, S):
    # split-K tiles are reduced in CTA order by the last contributor
    # (csrc/tc_pass2.cu): repeated launches -- single and paired -- give
    # bit-identical outputs
    g = torch.Generator(device="cuda").manual_seed(3 * m + n)
    a = torch.rand(m, n, device="cuda", generator=g)
    A = DeviceMatrix(a)
    x = torch.randn(n, S, device="cuda", generator=g)
    w = torch.randn(m, S, device="cuda", generator=g)
    lib = _lib.load()
    outs = []
    for _ in range(40):
        y, z, y2, z2 = zeros((m, S)), zeros((n, S)), zeros((m, S)), zeros((n, S))
        assert lib.cnmf_pass_forward(A.ptr, m, n, A.lda, x.data_ptr(), S, y.data_ptr(), stream()) == 0
        assert lib.cnmf_pass_transpose(A.ptr, m, n, A.lda, w.data_ptr(), S, z.data_ptr(), stream()) == 0
        assert lib.cnmf_pass_pair(A.ptr, m, n, A.lda, x.data_ptr(), y2.data_ptr(), w.data_ptr(), z2.data_ptr(), S,
                                  stream()) == 0
        torch.cuda.synchronize()
        outs.append((y, z, y2, z2))
    yref = a.double() @ x.double()
    assert ((outs[0][0].double() - yref).abs().max() / yref.abs().max()).item() < 1e-5
    for o in outs[1:]:
        for u, v in zip(o, outs[0]):
            assert torch.equal(u, v)


@pytest.mark.parametrize("m,n,s", [(10000, 5000, 30), (4000, 3000, 30), (3000, 4000, 30), (300, 200, 30),
                                   (2500, 1300, 60)])
def test_paired_pass_matches_separate(m, n, s):
    # one launch computing Y = A X and Z = A^T W (both range finders' passes)
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n)
    a = torch.rand(m, n, device="cuda", generator=g)
    A = DeviceMatrix(a)
    S = 32 if s <= 32 else 64
    x = zeros((n, S))
    w = zeros((m, S))
    x[:, :s] = torch.randn(n, s, device="cuda", generator=g)
    w[:, :s] = torch.randn(m, s, device="cuda", generator=g)
    lib = _lib.load()
    yref = a.double() @ x.double()
    zref = a.double().t() @ w.double()
    for _ in range(6):
        y, z = zeros((m, S)), zeros((n, S))
        _lib.call("cnmf_pass_pair", A.ptr, m, n, A.lda, x.data_ptr(), y.data_ptr(), w.data_ptr(), z.data_ptr(), s,
                  stream())
        torch.cuda.synchronize()
        assert ((y.double() - yref).abs().max() / yref.abs().max()).item() < 1e-5
        assert ((z.double() - zref).abs().max() / zref.abs().max()).item() < 1e-5


def test_compression_repeatable():
    # split-K passes reduce with fp32 atomics (order varies run to run); the
    # signal subspace is stable far below the 1e-4 tolerance
    a = O.dense_lowrank(3000, 1500, 20, 0.01, seed=3).astype(np.float32)
    cfg = C.CompressionConfig(r=20, r_ov=10, w=4, seed=9)
    q1 = C.structured_compress(a, cfg).Q
    q2 = C.structured_compress(a, cfg).Q
    assert O.projector_distance(q1[:, :20], q2[:, :20]) < 1e-6


def test_admm_stream_matches_persistent():
    # the three-launch streaming iteration (csrc/admm_stream.cu, forced with
    # CNMF_ADMM_STREAM=1) against the persistent kernel on the same
    # compressed problem: same iterates up to fp64 summation order
    from paper_1505_04650_b200.nmf import compressed_problem, run_admm

    a = O.dense_lowrank(2000, 1001, 20, 0.01, seed=0).astype(np.float32)
    A = DeviceMatrix(torch.from_numpy(a).cuda())
    cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), 2000, 1001)
    left, right, core = compressed_problem(A, cfg)
    outs = []
    for force in ("0", "1"):
        os.environ["CNMF_ADMM_STREAM"] = force
        try:
            u, vt, it, tr = run_admm(core, left.panel, 2000, right.panel, 1001, cfg, 20, max_iter=100, tol=0.0)
        finally:
            os.environ.pop("CNMF_ADMM_STREAM", None)
        torch.cuda.synchronize()
        outs.append((u.cpu().numpy(), vt.cpu().numpy(), it, np.array(tr)))
    (u0, v0, i0, t0), (u1, v1, i1, t1) = outs
    assert i0 == i1 == 100
    assert np.abs(u0 - u1).max() <= 1e-6 * np.abs(u0).max()
    assert np.abs(v0 - v1).max() <= 1e-6 * np.abs(v0).max()
    assert np.allclose(t0, t1, rtol=1e-8)


def test_admm_stream_resume_and_tol_stop():
    # the streaming driver (core_x / core_y split, csrc/admm_stream.cu):
    # (1) one iteration per call (resume = 1, step_limit = 1: the on_iteration
    # path) ends in the same state as a single call; (2) a tolerance stop
    # happens at the persistent kernel's iteration with its xc, yc
    from paper_1505_04650_b200.nmf import compressed_problem, run_admm

    a = O.dense_lowrank(1500, 900, 20, 0.01, seed=2).astype(np.float32)
    A = DeviceMatrix(torch.from_numpy(a).cuda())
    cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), 1500, 900)
    left, right, core = compressed_problem(A, cfg)
    run = lambda **kw: run_admm(core, left.panel, 1500, right.panel, 900, cfg, 20, **kw)
    os.environ["CNMF_ADMM_STREAM"] = "1"
    try:
        u0, v0, i0, t0 = run(max_iter=30, tol=0.0)
        seen = []
        u1, v1, i1, t1 = run(max_iter=30, tol=0.0,
                             on_iteration=lambda k, u, du, vt, dvt, xc, yc: seen.append((k, xc.clone(), yc.clone())))
    finally:
        os.environ.pop("CNMF_ADMM_STREAM", None)
    torch.cuda.synchronize()
    assert i0 == i1 == 30 and [k for k, _, _ in seen] == list(range(30))
    assert torch.equal(u0, u1) and torch.equal(v0, v1) and t0 == t1  # bit-reproducible, resumed or not
    # a tolerance the persistent kernel crosses mid-run: the streaming driver
    # stops at the same iteration with the same state
    tol, itp = None, None
    for cand in 10.0 ** np.arange(6, -3, -0.5):
        up, vp, itp, _ = run(max_iter=200, tol=float(cand))
        if 3 < itp < 200:
            tol = float(cand)
            break
    assert tol is not None
    os.environ["CNMF_ADMM_STREAM"] = "1"
    try:
        us, vs, its, _ = run(max_iter=200, tol=tol)
    finally:
        os.environ.pop("CNMF_ADMM_STREAM", None)
    torch.cuda.synchronize()
    assert its == itp, (its, itp, tol)
    assert (us - up).abs().max().item() <= 1e-6 * up.abs().max().item()
    assert (vs - vp).abs().max().item() <= 1e-6 * vp.abs().max().item()


def test_admm_rank_above_32_matches_oracle():
    # r > 32 with s > 32 (the shape class of configs[4], r = 50) runs on the
    # streaming iteration; parity with the oracle at a size it finishes fast
    a = O.dense_lowrank(900, 700, 40, 0.01, seed=4).astype(np.float32)
    cfg = C.CompressionConfig(r=40, r_ov=10, w=2, seed=3)
    fp = C.nmf_admm(a, 40, cfg=cfg, max_iter=60, tol=1e-4)
    ref = O.admm(a, 40, cfg=O.Config(40, 10, 2, 3), max_iter=60, tol=1e-4)
    assert fp.iterations == ref.iterations
    assert abs(fp.rel_error - ref.rel_error) <= 1e-3 * ref.rel_error


def test_relative_error_matches(golden):
    got = C.relative_error(golden["admm_a"], golden["admm_comp_X"], golden["admm_comp_Y"])
    assert abs(got - golden["relerr"][0]) < 1e-6
    with pytest.raises(C.UndefinedMetricError):
        C.relative_error(np.zeros((4, 4)), np.ones((4, 2)), np.ones((2, 4)))


def test_errors_for_ranks_above_64():
    # relative_error / compression_error for 64 < r <= 128 (the residual
    # kernel's second instantiation): against fp64 numpy
    g = np.random.default_rng(5)
    a = np.abs(g.standard_normal((700, 90))) @ np.abs(g.standard_normal((90, 520))) + 0.01 * g.standard_normal((700, 520))
    a = np.maximum(a, 0.0).astype(np.float32)
    x = np.abs(g.standard_normal((700, 100)))
    y = np.abs(g.standard_normal((100, 520))) * 0.01
    a64 = a.astype(np.float64)
    want = np.linalg.norm(a64 - x @ y) / np.linalg.norm(a64)
    assert abs(C.relative_error(a, x, y) - want) <= 1e-5 * want
    cfg = C.CompressionConfig(r=70, r_ov=10, w=1, seed=4)
    basis = C.structured_compress(a, cfg)
    q = np.asarray(basis.Q, dtype=np.float64)
    assert q.shape[1] == 80
    want_c = np.linalg.norm(a64 - q @ (q.T @ a64))
    assert abs(C.compression_error(a, basis) - want_c) <= 1e-4 * max(want_c, 1e-3 * np.linalg.norm(a64))


def test_admm_validates():
    with pytest.raises(C.ArgumentError):
        C.nmf_admm(np.random.default_rng(0).uniform(size=(40, 30)), 2, penalty_u=0.0)


# ---------------------------------------------------------------------------
# nmf_admm(compressed=False): the uncompressed loop (csrc/admm_full.cu)

def _full_case(m=300, n=200, r=5, seed=3):
    a = O.dense_lowrank(m, n, r, 0.01, seed=seed).astype(np.float32)
    return a, C.CompressionConfig(r=r, r_ov=10, w=4, seed=7), O.Config(r, 10, 4, 7)


def test_admm_uncompressed_matches_oracle():
    a, cfg, ocfg = _full_case()
    res = C.nmf_admm(a, 5, compressed=False, cfg=cfg, max_iter=60)
    ref = O.admm(a.astype(np.float64), 5, compressed=False, cfg=ocfg, max_iter=60)
    assert res.iterations == ref.iterations == 60
    assert abs(res.rel_error - ref.rel_error) <= 1e-3 * ref.rel_error
    # the objective ||A - xc yc||^2 per iteration (nmf.py:362), evaluated as
    # ||A||^2 - 2 <yc^T, A^T xc> + <Gx, Gy> from the iteration's own fp32
    # products: absolute error ~1e-7 of ||A||^2 (3xTF32 and fp32 panels)
    na2 = float(np.sum(a.astype(np.float64) ** 2))
    assert np.abs(np.array(res.objective_trace) - np.array(ref.trace)).max() <= 1e-6 * na2
    # early iterates agree to the fp32 products' precision
    short = C.nmf_admm(a, 5, compressed=False, cfg=cfg, max_iter=5)
    sref = O.admm(a.astype(np.float64), 5, compressed=False, cfg=ocfg, max_iter=5)
    assert np.abs(short.X - sref.X).max() <= 1e-4 * max(1.0, np.abs(sref.X).max())
    assert np.abs(short.Y - sref.Y).max() <= 1e-4 * max(1.0, np.abs(sref.Y).max())
    assert short.X.min() >= 0 and short.Y.min() >= 0


def test_admm_uncompressed_tol_stop_and_callback():
    a, cfg, ocfg = _full_case(seed=5)
    probe = O.admm(a.astype(np.float64), 5, compressed=False, cfg=ocfg, max_iter=30, tol=0.0)
    tol = probe.scores[12] * (1 + 1e-3)  # first reached at iteration <= 12
    ref = O.admm(a.astype(np.float64), 5, compressed=False, cfg=ocfg, max_iter=30, tol=tol)
    seen = []
    res = C.nmf_admm(a, 5, compressed=False, cfg=cfg, max_iter=30, tol=tol,
                     on_iteration=lambda k, st: seen.append((k, np.array(st.u))))
    assert res.iterations == ref.iterations < 30
    assert [k for k, _ in seen] == list(range(res.iterations))
    plain = C.nmf_admm(a, 5, compressed=False, cfg=cfg, max_iter=30, tol=tol)
    assert plain.iterations == res.iterations
    assert np.abs(seen[-1][1] - res.X).max() == 0.0


def test_admm_uncompressed_limits():
    a, cfg, _ = _full_case(m=100, n=80, r=5)
    with pytest.raises(C.ArgumentError):
        C.nmf_admm(a, 40, compressed=False, cfg=C.CompressionConfig(r=40, r_ov=10, w=4, seed=1))
    res = C.nmf_admm(a, 5, compressed=False, cfg=cfg, max_iter=0)
    assert res.iterations == 0


# ------------------------------------------------- API completeness -----

def test_compression_error_spectral_matches_power_iteration():
    # compress.py:250-286: the spectral norm of A - Q Q^T A by the reference's
    # seeded power iteration (the exact 2-norm as the yardstick)
    a = O.dense_lowrank(900, 700, 8, 0.05, seed=4).astype(np.float32).astype(np.float64)
    basis = C.structured_compress(a, C.CompressionConfig(r=8, r_ov=4, w=2, seed=1))
    q = basis.Q
    resid = a - q @ (q.T @ a)
    got = C.compression_error(a, basis, norm="spectral")
    assert abs(got - np.linalg.norm(resid, 2)) <= 1e-3 * np.linalg.norm(resid, 2)
    fro = C.compression_error(a, basis)
    assert abs(fro - np.linalg.norm(resid)) <= 1e-4 * np.linalg.norm(resid)
    with pytest.raises(C.ArgumentError):
        C.compression_error(a, basis, norm="nuclear")


def test_canonical_qr_matches_reference_convention():
    # compress.py:136-145: reduced QR with diag(R) >= 0
    b = np.random.default_rng(3).standard_normal((2000, 37))
    q, r = C.canonical_qr(b)
    qr_, rr = O.qr_pos(b)
    assert np.all(np.diag(r) > 0)
    assert np.abs(q - qr_).max() < 1e-5
    assert np.abs(r - rr).max() < 1e-5 * np.abs(rr).max()
    assert np.allclose(np.tril(r, -1), 0.0)


def test_kkt_residual_matches_oracle():
    # nmf.py:246-303 at an ADMM state delivered by on_iteration
    d = O.dense_lowrank(300, 200, 4, 0.01, seed=8)
    states = []
    C.nmf_admm(d, 4, cfg=C.CompressionConfig(r=4, seed=2), max_iter=5, tol=0.0,
               on_iteration=lambda k, st: states.append(st))
    st = states[-1]
    cfg = O.adjust(O.Config(4, 10, 4, 2), *d.shape)
    left, right = O.compressed_bases(d, cfg)
    core = (left.T @ d) @ right.T
    got = C.kkt_residual(st, core, left, right)
    ref = O.kkt(st.xc, st.yc, st.u, st.v, st.dual_u, st.dual_v, core, left, right)
    np.testing.assert_allclose([got.grad_left, got.grad_right, got.feas_left, got.feas_right, got.comp_left,
                                got.comp_right], ref, rtol=1e-6, atol=1e-9)
    assert got.max_residual == max(ref) or abs(got.max_residual - max(ref)) <= 1e-6 * max(ref)


# --------------------------------------------------------- fp64 path -----

def test_fp64_range_finder_matches_reference_golden(golden):
    # precision="fp64" (configs[0] is an fp64 workload): the reference's own
    # reorthogonalized basis to fp64 accuracy, columns included
    a = golden["cmp_a"]
    cfg = C.CompressionConfig(r=8, r_ov=12, w=2, seed=3)
    q = C.structured_compress(a, cfg, precision="fp64").Q
    ref = golden["cmp_q_w2_reorth"]
    assert O.projector_distance(q, ref) < 1e-9
    assert np.abs(q - ref).max() < 1e-8
    qr_ = C.structured_compress_rows(a, cfg, precision="fp64").Q
    assert O.projector_distance(qr_, golden["cmp_qrows_w2_reorth"]) < 1e-9


@pytest.mark.parametrize("sel", ["spa", "xray"])
def test_fp64_snmf_config0_shape(sel):
    a, truth = O.near_separable(500, 2000, 10, 1.0, 0.01, seed=11)
    cfg = C.CompressionConfig(r=10, r_ov=10, w=4, seed=2)
    res = C.snmf(a, 10, selector=sel, cfg=cfg, precision="fp64")
    ref = O.snmf(a, 10, selector=sel, cfg=O.Config(10, 10, 4, 2))
    assert np.array_equal(res.K, ref.K)
    assert abs(res.rel_error_full - ref.rel_error_full) <= 1e-9 * ref.rel_error_full
    assert abs(res.rel_error_reduced - ref.rel_error_reduced) <= 1e-8 * max(ref.rel_error_reduced, 1e-12)
    assert np.abs(res.Y - ref.Y).max() <= 1e-8 * max(1.0, np.abs(ref.Y).max())


@pytest.mark.parametrize("r,noise", [(50, 0.25), (20, 0.4), (50, 0.01)])
def test_residual_pass_path(r, noise):
    # ||A - X Y|| through one tensor-core forward pass (||A||^2 - 2 <A Y^T, X> +
    # <X^T X, Y Y^T>) against an fp64 reference; small residuals (noise 0.01:
    # rel ~ 1e-2, too much cancellation) must take the direct kernel
    from paper_1505_04650_b200.nmf import _rel_error

    m, n = 9000, 8000  # m n >= 2^26: the pass path is eligible
    g = torch.Generator(device="cuda").manual_seed(r)
    x = torch.rand(m, r, device="cuda", dtype=torch.float64, generator=g)
    y = torch.rand(r, n, device="cuda", dtype=torch.float64, generator=g)
    a = (x @ y) * (1.0 + noise * torch.randn(m, n, device="cuda", dtype=torch.float64, generator=g))
    a32 = a.clamp_(min=0).float()
    ref = float(torch.linalg.norm(a32.double() - x @ y) / torch.linalg.norm(a32.double()))
    A = DeviceMatrix(a32)
    vt = y.t().contiguous()
    got = {}
    for mode in ("1", "0"):
        os.environ["CNMF_RESID_PASS"] = mode
        try:
            got[mode] = _rel_error(A, x, vt)
        finally:
            os.environ.pop("CNMF_RESID_PASS", None)
    # the direct kernel forms X Y from fp32 factors in FP32 FMA: ~1e-5 relative
    assert abs(got["0"] - ref) <= 2e-5 * ref, (got, ref)
    assert abs(got["1"] - ref) <= 2e-5 * ref, (got, ref)
