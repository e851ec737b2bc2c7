"""Full-size parity at the BASELINE.json shapes, against fixtures written by
running the REFERENCE itself (tests/golden/make_golden_large.py; the
matrices are regenerated here from the same numpy seeds).

* configs[1] shape (and a 2000 x 1000 cut): the full 30-column compressed
  subspace must agree with the reference's reorthogonalized basis within the
  north-star projector distance of 1e-4 (measured 7.0e-5 .. 8.6e-5; for
  scale, the reference's OWN basis moves 5.4e-5 .. 6.4e-5 when A is perturbed
  by one fp32 rounding, 2^-24 relative: stored in the fixture).
* configs[2] at its full 2,000,000 x 200: the SPA picks are bit-exact (pick
  order included). Whether the NNLS right factor (absolute tolerance 1e-10
  on gradients of size ~1e6) trips the reference's exchange cap is decided by
  rounding: the reference itself returns for some 2^-24 perturbations of A
  and raises for others (fixture), so either outcome is the reference's.
"""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from oracle import cnmf_oracle as O  # noqa: E402
from make_golden_large import dense_config1, proj_dist  # noqa: E402

import paper_1505_04650_b200 as C  # noqa: E402

FIX = os.path.join(ROOT, "tests", "golden", "reference_large.npz")


@pytest.fixture(scope="module")
def large():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return np.load(FIX)


@pytest.mark.parametrize("m,n", [(2000, 1000), (10000, 5000)])
def test_compress_config1_shape_full_subspace(large, m, n):
    a = dense_config1(m, n, seed=11).astype(np.float32)
    q = C.structured_compress(a, C.CompressionConfig(r=20, r_ov=10, w=4, seed=3)).Q
    key = f"c1_{m}x{n}"
    ref = large[key + "_q"].astype(np.float64)
    band = float(large[key + "_band"].max())
    d = proj_dist(ref, q)
    print(f"{key}: projector distance {d:.3e}, reference band {band:.3e}")
    assert np.linalg.norm(q.T @ q - np.eye(30)) < 1e-5
    assert d <= 1e-4, (d, band)  # north_star's bound as stated (band: the reference's own movement)
    # the stock (reorthogonalize=False) reference basis is a different
    # subspace altogether ("reorthogonalize")
    assert float(large[key + "_stock_dist"]) > 0.9


@pytest.mark.parametrize("seed", [1, 2])
def test_snmf_config2_fullsize_picks(large, seed):
    a, truth = O.near_separable(2_000_000, 200, 20, 0.5, 0.005, seed=seed)
    a = a.astype(np.float32)
    assert np.array_equal(np.asarray(truth), large[f"c2_seed{seed}_truth"])
    cfg = C.CompressionConfig(r=20, r_ov=10, w=2, seed=7)
    try:
        res = C.snmf(a, 20, selector="spa", cfg=cfg)
        picks, returned = res.K, True
    except C.ConvergenceError as e:
        picks, returned = e.picks, False
    assert np.array_equal(picks, large[f"c2_seed{seed}_picks"])
    outcomes = large[f"c2_seed{seed}_nnls_returns"]
    # the reference's own outcome under 2^-24 perturbations includes ours
    assert (1 if returned else 0) in set(outcomes.tolist()) or outcomes.min() != outcomes.max()
    if returned:
        assert res.rel_error_full < 0.01


FIX4 = os.path.join(ROOT, "tests", "golden", "reference_c4.npz")


def classical_config4(m, n, seed):
    """configs[4] generator at reduced size (tests/golden/make_golden_c4.py)."""
    g = np.random.default_rng(seed)
    x = g.uniform(size=(m, 50))
    y = g.uniform(size=(50, n))
    y *= g.uniform(size=(50, n)) >= 0.7
    return np.maximum(x @ y + 0.01 * g.standard_normal((m, n)), 0.0)


@pytest.mark.parametrize("m,n", [(4000, 2000), (12000, 6000)])
def test_compress_config4_shape_full_subspace(m, n):
    # S = 64 panels (r = 50, s = 60): the 256-row-unit pass kernel's wide
    # configuration, against the reference's reorthogonalized basis
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    fx = np.load(FIX4)
    a = classical_config4(m, n, seed=13).astype(np.float32)
    q = C.structured_compress(a, C.CompressionConfig(r=50, r_ov=10, w=4, seed=3)).Q
    key = f"c4_{m}x{n}"
    ref = fx[key + "_q"].astype(np.float64)
    band = float(fx[key + "_band"].max())
    d = proj_dist(ref, q)
    print(f"{key}: projector distance {d:.3e}, reference band {band:.3e}")
    assert np.linalg.norm(q.T @ q - np.eye(60)) < 1e-5
    assert d <= 1e-4, (d, band)  # north_star's bound as stated (band: the reference's own movement)
