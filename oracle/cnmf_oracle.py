"""CPU oracle for the compressed-NMF hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference package
(``/root/reference/pkg/src/cnmf``) for the functions on the hot path. It is
the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product (``paper_1505_04650_b200``) never imports or calls it and fails
loudly when its CUDA library is missing.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against fixtures produced by running the reference itself
(``tests/golden/make_golden.py``), and the Gaussian test matrix is checked
bit-for-bit against numpy's Philox/ziggurat stream, the reference's own
RNG (rng.py:38-70).

Every function cites the reference file:line it restates.
"""

from dataclasses import dataclass, replace

import numpy as np

MASK64 = (1 << 64) - 1
OMEGA_CHUNK = 4096            # compress.py:22
POWER_NORM_SEED = 0x5EC7AA1   # compress.py:23
RIDGE_SCALE = 1e-12           # nnls.py:17
ZERO_CLIP = 1e-14             # nnls.py:18
RANK_TOL = 1e-14              # snmf.py:22
TINY = np.finfo(np.float64).tiny


class OracleError(Exception):
    """Raised where the reference raises; ``kind`` names the reference class."""

    def __init__(self, kind, message, **extra):
        super().__init__(message)
        self.kind = kind
        self.__dict__.update(extra)


# ----------------------------------------------------------------------------
# RNG (rng.py)
# ----------------------------------------------------------------------------

def fnv1a64(tag):
    """FNV-1a over UTF-8 bytes (rng.py:23-28)."""
    h = 0xCBF29CE484222325
    for b in tag.encode("utf-8"):
        h = ((h ^ b) * 0x100000001B3) & MASK64
    return h


def splitmix64(x):
    """SplitMix64 finalizer (rng.py:31-35)."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def child_seed(seed, tag):
    """Child stream seed (rng.py:56-58, rng.py:73-75)."""
    return splitmix64((int(seed) & MASK64) ^ fnv1a64(tag))


def generator(seed):
    """numpy Philox(4x64) generator keyed by the 64-bit seed (rng.py:49-51)."""
    return np.random.Generator(np.random.Philox(key=int(seed) & MASK64))


def test_matrix(rows, cols, seed):
    """Seeded Gaussian test matrix drawn in 4096-row chunks, one child stream
    per chunk (compress.py:115-127)."""
    base = child_seed(seed, "omega")
    parts = []
    for c, lo in enumerate(range(0, rows, OMEGA_CHUNK)):
        hi = min(lo + OMEGA_CHUNK, rows)
        parts.append(generator(child_seed(base, f"chunk{c}")).standard_normal((hi - lo, cols)))
    return np.vstack(parts)


def uniform_matrix(seed, tag, shape):
    """``Rng(seed).child(tag).uniform(shape)`` (rng.py:63-64, nmf.py:186-188)."""
    return generator(child_seed(seed, tag)).uniform(0.0, 1.0, size=shape)


# ----------------------------------------------------------------------------
# Compression (compress.py)
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class Config:
    """CompressionConfig (compress.py:27-51)."""

    r: int
    r_ov: int = 10
    w: int = 4
    seed: int = 0

    @property
    def width(self):
        return self.r + self.r_ov


def adjust(cfg, m, n):
    """Basis-width rule min(max(20, r + r_ov), n, m) (compress.py:101-112)."""
    if cfg.r >= min(m, n):
        raise OracleError("InfeasibleRankError", "rank infeasible")
    width = min(max(20, cfg.r + cfg.r_ov), n, m)
    return replace(cfg, r_ov=width - cfg.r)


def qr_pos(b):
    """Reduced QR with nonnegative diag(R) (compress.py:136-145)."""
    q, r = np.linalg.qr(b)
    sgn = np.sign(np.diag(r))
    sgn[sgn == 0] = 1.0
    return q * sgn, sgn[:, None] * r


def range_basis(a, cfg, reorth=True):
    """Randomized range finder with w power passes (compress.py:156-199).

    ``reorth`` mirrors the reference's ``reorthogonalize`` flag. Both settings
    define the same Q in exact arithmetic (the intermediate QRs right-multiply
    the sketch by upper-triangular factors, which preserves every leading
    column span); the oracle defaults to the numerically stable one.
    """
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    if cfg.width > min(m, n):
        raise OracleError("InfeasibleRankError", "basis width exceeds min(m, n)")
    b = a @ test_matrix(n, cfg.width, cfg.seed)
    for _ in range(cfg.w):
        if reorth:
            b = qr_pos(b)[0]
        c = a.T @ b
        if reorth:
            c = qr_pos(c)[0]
        b = a @ c
    if not np.isfinite(b).all():
        raise OracleError("NumericError", "non-finite sketch")
    return qr_pos(b)[0]


def row_basis(a, cfg, reorth=True):
    """Row-space basis = range basis of A^T (compress.py:202-212)."""
    return range_basis(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T), cfg, reorth)


def residual_norm(a, q):
    """||A - Q Q^T A||_F (compress.py:250-262)."""
    return float(np.linalg.norm(a - q @ (q.T @ a)))


def gaussian_basis(m, s, seed):
    """Q = s^-1/2 * Gaussian (compress.py:238-247)."""
    g = generator(child_seed(seed, "gaussian-projection")).standard_normal((m, s))
    return g / np.sqrt(s)


def projector_distance(q1, q2):
    """||Q1 Q1^T - Q2 Q2^T||_2 for orthonormal Q1, Q2 of equal width (the
    north-star parity metric) = sine of the largest principal angle, computed
    as ||Q2 - Q1 (Q1^T Q2)||_2 (accurate for small angles)."""
    q1 = np.asarray(q1, dtype=np.float64)
    q2 = np.asarray(q2, dtype=np.float64)
    if q1.shape != q2.shape:
        return 1.0
    return float(np.linalg.norm(q2 - q1 @ (q1.T @ q2), 2))


def dominant_subspace(q, a, k):
    """Orthonormal basis of the top-k left singular subspace of Q Q^T A: the
    numerically determined part of a range basis on low-rank + noise data."""
    u = np.linalg.svd(q.T @ a, full_matrices=False)[0][:, :k]
    return q @ u


# ----------------------------------------------------------------------------
# NNLS (nnls.py)
# ----------------------------------------------------------------------------

def nnls(c, d, tol=1e-10, max_exchanges=None):
    """Active-set NNLS, column by column (nnls.py:21-111, nnls.py:122-168).

    The reference advances all columns in lockstep; the per-column arithmetic
    is identical, so the oracle walks one column at a time.
    """
    c = np.asarray(c, dtype=np.float64)
    vec = np.ndim(d) == 1
    d = np.asarray(d, dtype=np.float64).reshape(c.shape[0], -1)
    q, k = c.shape[1], d.shape[1]
    cap = max_exchanges if max_exchanges is not None else 3 * q
    gram = c.T @ c
    target = c.T @ d
    ridge = RIDGE_SCALE * float(np.trace(gram))
    h = np.zeros((q, k))
    for j in range(k):
        h[:, j] = _nnls_column(gram, target[:, j], tol, cap, ridge)
    np.maximum(h, 0.0, out=h)
    return h[:, 0] if vec else h


def _solve_support(gram, t, pas, ridge):
    q = gram.shape[0]
    mat = gram * np.outer(pas, pas)
    mat[np.arange(q), np.arange(q)] += ~pas
    rhs = np.where(pas, t, 0.0)
    try:
        z = np.linalg.solve(mat, rhs)
        if not np.isfinite(z).all():
            raise np.linalg.LinAlgError
    except np.linalg.LinAlgError:
        mat[np.arange(q), np.arange(q)] += ridge * pas
        z = np.linalg.solve(mat, rhs)
    return z


def _nnls_column(gram, t, tol, cap, ridge):
    q = gram.shape[0]
    h = np.zeros(q)
    pas = np.zeros(q, dtype=bool)
    grad = t.copy()
    swaps = 0
    while True:
        cand = np.where(pas, -np.inf, grad)
        i = int(np.argmax(cand))
        if cand[i] <= tol:
            break
        pas[i] = True
        swaps += 1
        if swaps > cap:
            raise OracleError("ConvergenceError", "exchange cap exceeded")
        while True:
            z = _solve_support(gram, t, pas, ridge)
            if ((z > 0) | ~pas).all():
                h = z
                break
            # step back towards z until a passive coordinate hits zero (nnls.py:151-168)
            blk = pas & (z <= 0)
            den = h[blk] - z[blk]
            ratio = np.where(den > 0, h[blk] / np.where(den > 0, den, 1.0), 0.0)
            alpha = float(ratio.min()) if ratio.size else 0.0
            h = h + alpha * (z - h)
            scale = max(float(np.max(np.abs(h))), 1.0)
            rel = blk & (h <= ZERO_CLIP * scale)
            if not rel.any():
                rel = np.zeros(q, dtype=bool)
                rel[np.flatnonzero(blk)[int(np.argmin(ratio))]] = True
            h[rel] = 0.0
            pas[rel] = False
            swaps += 1
            if swaps > cap:
                raise OracleError("ConvergenceError", "exchange cap exceeded")
        grad = t - gram @ h
    return h


# ----------------------------------------------------------------------------
# Separable NMF (snmf.py)
# ----------------------------------------------------------------------------

def spa(rm, r):
    """Successive projection (snmf.py:39-71); ties -> lowest index."""
    w = np.array(rm, dtype=np.float64, copy=True)
    s, n = w.shape
    if not 1 <= r <= min(s, n):
        raise OracleError("ArgumentError", "bad r")
    sq = np.einsum("ij,ij->j", w, w)
    floor = (np.sqrt(sq.max()) * RANK_TOL) ** 2
    picks = []
    for _ in range(r):
        j = int(np.argmax(sq))
        if sq[j] <= floor:
            raise OracleError("RankDeficiencyError", "deficient", picks=list(picks))
        picks.append(j)
        v = w[:, j] / np.sqrt(sq[j])
        w -= np.outer(v, v @ w)
        sq = np.einsum("ij,ij->j", w, w)
        sq[picks] = 0.0
    return np.asarray(picks, dtype=np.int64)


def xray(rm, r, mass=None, nnls_tol=1e-10):
    """Greedy residual-driven extreme columns with NNLS refits (snmf.py:74-126)."""
    full = np.asarray(rm, dtype=np.float64)
    s, n = full.shape
    if not 1 <= r <= min(s, n):
        raise OracleError("ArgumentError", "bad r")
    if mass is None:
        if full.min() >= 0:
            mass = np.ones(s)
        else:
            nrm = np.sqrt(np.einsum("ij,ij->j", full, full))
            keep = nrm > 0
            mass = (full[:, keep] / nrm[keep]).sum(axis=1)
    denom = mass @ full
    ok = denom > RANK_TOL * max(float(np.abs(denom).max()), 1.0)
    res = full.copy()
    floor = (np.sqrt(np.einsum("ij,ij->j", full, full).max()) * RANK_TOL) ** 2
    picks = []
    for _ in range(r):
        sq = np.einsum("ij,ij->j", res, res)
        sq[picks] = 0.0
        j = int(np.argmax(sq))
        if sq[j] <= floor:
            raise OracleError("RankDeficiencyError", "deficient", picks=list(picks))
        score = np.where(ok, (res[:, j] @ full) / np.where(ok, denom, 1.0), -np.inf)
        score[picks] = -np.inf
        i = int(np.argmax(score))
        if not np.isfinite(score[i]):
            raise OracleError("RankDeficiencyError", "no scorable column", picks=list(picks))
        picks.append(i)
        coef = nnls(full[:, picks], full, tol=nnls_tol)
        res = full - full[:, picks] @ coef
    return np.asarray(picks, dtype=np.int64)


@dataclass
class SnmfOut:
    K: np.ndarray
    Y: np.ndarray
    rel_error_reduced: float
    rel_error_full: float
    reduced: np.ndarray
    mass: np.ndarray


def snmf(a, r, selector="spa", cfg=None, nnls_tol=1e-10, reorth=True, basis=None):
    """Compressed separable NMF pipeline (snmf.py:154-232, reduction="compressed")."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    cfg = adjust(cfg or Config(r=r, r_ov=10, w=0, seed=0), m, n)
    q = range_basis(a, cfg, reorth) if basis is None else basis
    red = q.T @ a
    mass = q.sum(axis=0)
    picks = spa(red, r) if selector == "spa" else xray(red, r, mass=mass, nnls_tol=nnls_tol)
    y = nnls(red[:, picks], red, tol=nnls_tol)
    rel_red = float(np.linalg.norm(red - red[:, picks] @ y)) / float(np.linalg.norm(red))
    rel_full = float(np.linalg.norm(a - a[:, picks] @ y) / np.linalg.norm(a))
    return SnmfOut(picks, y, rel_red, rel_full, red, mass)


# ----------------------------------------------------------------------------
# ADMM NMF (nmf.py:226-377)
# ----------------------------------------------------------------------------

def rel_error(a, x, y):
    """||A - X Y||_F / ||A||_F (nmf.py:53-75)."""
    return float(np.linalg.norm(a - x @ y) / np.linalg.norm(a))


def kkt(xc, yc, u, v, du, dv, core, left, right):
    """Six KKT residual norms (nmf.py:281-303); left/right None = identity."""
    lm = (lambda z: z) if left is None else (lambda z: left @ z)
    ltm = (lambda z: z) if left is None else (lambda z: left.T @ z)
    rm = (lambda z: z) if right is None else (lambda z: z @ right)
    rtm = (lambda z: z) if right is None else (lambda z: z @ right.T)
    e = xc @ yc - core
    out = (
        np.linalg.norm(e @ yc.T + ltm(du)),
        np.linalg.norm(xc.T @ e + rtm(dv)),
        np.linalg.norm(lm(xc) - u),
        np.linalg.norm(rm(yc) - v),
        np.sqrt(np.sum((du * u) ** 2) + np.sum(np.maximum(du, 0) ** 2) + np.sum(np.maximum(-u, 0) ** 2)),
        np.sqrt(np.sum((dv * v) ** 2) + np.sum(np.maximum(dv, 0) ** 2) + np.sum(np.maximum(-v, 0) ** 2)),
    )
    return tuple(float(x) for x in out)


@dataclass
class AdmmOut:
    X: np.ndarray
    Y: np.ndarray
    iterations: int
    trace: list
    scores: list
    rel_error: float
    left: np.ndarray
    right: np.ndarray


def compressed_bases(a, cfg, reorth=True):
    """Left basis L (m x s) and right basis R (s x n) (nmf.py:120-135)."""
    lcfg = replace(cfg, seed=child_seed(cfg.seed, "left-basis"))
    rcfg = replace(cfg, seed=child_seed(cfg.seed, "right-basis"))
    return range_basis(a, lcfg, reorth), row_basis(a, rcfg, reorth).T


def admm(a, r, compressed=True, cfg=None, pu=1.0, pv=1.0, step=1.0, max_iter=500,
         tol=1e-4, reorth=True, bases=None, on_iteration=None):
    """ADMM on U = L Xc, V = Yc R, U, V >= 0 (nmf.py:306-377)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if cfg is None:
        cfg = Config(r=r, r_ov=10, w=4, seed=0)
    if compressed:
        cfg = adjust(cfg, m, n)
        left, right = bases if bases is not None else compressed_bases(a, cfg, reorth)
        core = (left.T @ a) @ right.T
    else:
        left = right = None
        core = a
    u, v, it, trace, scores = admm_compressed(core, left, right, m, n, r, cfg, pu, pv, step, max_iter, tol,
                                              on_iteration)
    return AdmmOut(u, v, it, trace, scores, rel_error(a, u, v), left, right)


def admm_compressed(core, left, right, m, n, r, cfg, pu=1.0, pv=1.0, step=1.0, max_iter=500, tol=1e-4,
                    on_iteration=None):
    """The ADMM loop of nmf.py:334-377 given the compressed problem (core =
    L^T A R^T, left L m x s, right R s x n; None for the uncompressed case)."""
    u = uniform_matrix(cfg.seed, "init-left", (m, r))
    v = uniform_matrix(cfg.seed, "init-right", (r, n))
    du = np.zeros((m, r))
    dv = np.zeros((r, n))
    yc = v if right is None else v @ right.T
    eye = np.eye(r)
    lm = (lambda z: z) if left is None else (lambda z: left @ z)
    ltm = (lambda z: z) if left is None else (lambda z: left.T @ z)
    rm = (lambda z: z) if right is None else (lambda z: z @ right)
    rtm = (lambda z: z) if right is None else (lambda z: z @ right.T)
    trace, scores, it = [], [], 0
    for k in range(max_iter):
        rhs = core @ yc.T + pu * ltm(u) - ltm(du)
        xc = np.linalg.solve(yc @ yc.T + pu * eye, rhs.T).T
        yc = np.linalg.solve(xc.T @ xc + pv * eye, xc.T @ core + pv * rtm(v) - rtm(dv))
        lx, ry = lm(xc), rm(yc)
        u = np.maximum(lx + du / pu, 0.0)
        v = np.maximum(ry + dv / pv, 0.0)
        du = du + step * pu * (lx - u)
        dv = dv + step * pv * (ry - v)
        it = k + 1
        trace.append(float(np.sum((core - xc @ yc) ** 2)))
        if on_iteration is not None:
            on_iteration(k, (xc, yc, u, v, du, dv))
        score = max(kkt(xc, yc, u, v, du, dv, core, left, right))
        scores.append(score)
        if score < tol:
            break
        if k >= 50 and score > 10.0 * scores[k - 50]:
            raise OracleError("DivergenceError", "diverging", trace=scores)
    return u, v, it, trace, scores


# ----------------------------------------------------------------------------
# Synthetic inputs named by BASELINE.json configs (seeded; not the
# reference's generators, which the bench configs do not use)
# ----------------------------------------------------------------------------

def near_separable(m, n, r, alpha, noise, seed):
    """W ~ |N(0,1)|, H = [I_r | Dirichlet(alpha)] permuted, A = max(W H + noise, 0)."""
    g = np.random.default_rng(seed)
    w = np.abs(g.standard_normal((m, r)))
    h = np.zeros((r, n))
    h[:, :r] = np.eye(r)
    h[:, r:] = g.dirichlet(np.full(r, alpha), size=n - r).T
    perm = g.permutation(n)
    h = h[:, perm]
    truth = np.sort(np.flatnonzero(perm < r))
    a = np.maximum(w @ h + noise * g.standard_normal((m, n)), 0.0)
    return a, truth


def dense_lowrank(m, n, r, noise, seed):
    """X, Y ~ U[0,1], A = max(X Y + noise, 0) (BASELINE.json configs[1])."""
    g = np.random.default_rng(seed)
    x = g.uniform(size=(m, r))
    y = g.uniform(size=(r, n))
    return np.maximum(x @ y + noise * g.standard_normal((m, n)), 0.0)
