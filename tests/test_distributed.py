"""Column-sharded driver (paper_1505_04650_b200/distributed.py) on CPU: two
gloo ranks, each holding one column shard, with the oracle's numpy
arithmetic standing in for the device kernels. The collectives and the
shard bookkeeping are the product code; the results must equal the
single-process oracle on the full matrix."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import cnmf_oracle as O  # noqa: E402
from paper_1505_04650_b200 import distributed as D  # noqa: E402
from paper_1505_04650_b200.compress import CompressionConfig, adjust_config  # noqa: E402


class Shard:
    """The local column block, shaped like DeviceMatrix (m, n attributes)."""

    def __init__(self, a):
        self.a = np.ascontiguousarray(a)
        self.m, self.n = a.shape


class NumpyOps:
    """Test double of DeviceOps: fp64 numpy arithmetic from the oracle."""

    def panel_ld(self, s):
        return 32 if s <= 32 else 64 if s <= 64 else 128

    def begin(self, s):
        pass

    def end(self):
        pass

    def zeros(self, shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=torch.float64)

    def omega_rows(self, seed, row0, rows, s, S):
        out = self.zeros((rows, S))
        ch = O.OMEGA_CHUNK
        for c in range(row0 // ch, (row0 + rows - 1) // ch + 1):
            start, end = c * ch, min(row0 + rows, (c + 1) * ch)
            blk = O.generator(O.child_seed(seed, f"chunk{c}")).standard_normal((end - start, s))
            lo = max(row0, start)
            out[lo - row0: end - row0, :s] = torch.from_numpy(blk[lo - start:])
        return out

    def forward(self, A, X, S):
        return torch.from_numpy(A.a @ X.numpy())

    def transpose(self, A, W, S):
        return torch.from_numpy(np.ascontiguousarray(A.a.T @ W.numpy()))

    def orthonormalize(self, P, s):
        P[:, :s] = torch.from_numpy(O.qr_pos(P[:, :s].numpy())[0])
        return P

    def cross(self, P1, P2, S):
        return P1.t() @ P2

    def cholesky_inverse(self, G, s, S):
        g = G[:s, :s].numpy()
        R = np.linalg.cholesky(np.triu(g) + np.triu(g, 1).T).T
        T = self.zeros((S, S))
        T[:s, :s] = torch.from_numpy(np.linalg.inv(R))
        G.zero_()
        return T

    def apply(self, P, T, S):
        P.copy_(P @ T)
        return P

    def residual(self, A, X, Yt):
        d = A.a - X.numpy() @ Yt.numpy().T
        return torch.tensor([float((d * d).sum()), float((A.a * A.a).sum())], dtype=torch.float64)

    # ---- sharded ADMM: the phases of nmf.py:334-377 in numpy ----
    def uniform(self, seed, start, rows, cols, transpose=False):
        g = O.generator(seed)
        g.bit_generator.advance(start // 4)
        g.bit_generator.random_raw(start % 4)
        x = g.uniform(0.0, 1.0, size=(rows, cols))
        return torch.from_numpy(np.ascontiguousarray(x.T) if transpose else x)

    def admm_shard_begin(self, s, r, GL, GR):
        return {"s": s, "r": r, "k": 0, "done": 0, "iters": 0, "div": -1,
                "sums": torch.zeros(2 * (2 * s * r + 4), dtype=torch.float64), "xc": None, "yc": None}

    def admm_shard_sweep(self, st, L, Rt, u, du, vt, dvt, s, r, pu, pv, step, update):
        if update and st["done"]:
            return st["sums"]
        out = []
        for P, x, dx, z, pen in ((L, u, du, st["xc"], pu), (Rt, vt, dvt, None if st["yc"] is None else st["yc"].T, pv)):
            Pn = P[:, :s].numpy()
            if update:
                lx = Pn @ z
                xn = np.maximum(lx + dx.numpy() / pen, 0.0)
                dxn = dx.numpy() + step * pen * (lx - xn)
                x.copy_(torch.from_numpy(xn))
                dx.copy_(torch.from_numpy(dxn))
                kkt = [float(((lx - xn) ** 2).sum()), float(((dxn * xn) ** 2).sum()),
                       float((np.maximum(dxn, 0) ** 2).sum()), float((np.maximum(-xn, 0) ** 2).sum())]
            else:
                kkt = [0.0] * 4
            out += [(Pn.T @ x.numpy()).ravel(), (Pn.T @ dx.numpy()).ravel(), np.array(kkt)]
        st["sums"].copy_(torch.from_numpy(np.concatenate(out)))
        return st["sums"]

    def admm_shard_core(self, st, core, xc, yc, s, r, pu, pv, step, tol, trace, scores, k, max_iter, first, solve):
        if st["done"]:
            return
        sr, ln = s * r, 2 * s * r + 4
        sm = st["sums"].numpy()
        lu, ldu, lk = sm[:sr].reshape(s, r), sm[sr:2 * sr].reshape(s, r), sm[2 * sr:ln]
        rv, rdv, rk = sm[ln:ln + sr].reshape(s, r), sm[ln + sr:ln + 2 * sr].reshape(s, r), sm[ln + 2 * sr:]
        cm = core.numpy()
        if first:
            st["yc"] = rv.T.copy()
        elif k > 0:
            x_, y_ = st["xc"], st["yc"]
            e = x_ @ y_ - cm
            sc = max(np.linalg.norm(e @ y_.T + ldu), np.linalg.norm(x_.T @ e + rdv.T), np.sqrt(lk[0]),
                     np.sqrt(rk[0]), np.sqrt(lk[1] + lk[2] + lk[3]), np.sqrt(rk[1] + rk[2] + rk[3]))
            trace[k - 1] = float((e * e).sum())
            scores[k - 1] = sc
            st["k"] = k
            if sc < tol or k >= max_iter:
                st["done"], st["iters"] = 1, k
                return
            if k - 1 >= 50 and sc > 10.0 * float(scores[k - 51]):
                st["div"], st["done"], st["iters"] = k - 1, 1, k
                return
        if not solve or k >= max_iter:
            return
        eye = np.eye(r)
        y_ = st["yc"]
        x_ = np.linalg.solve(y_ @ y_.T + pu * eye, (cm @ y_.T + pu * lu - ldu).T).T
        y_ = np.linalg.solve(x_.T @ x_ + pv * eye, x_.T @ cm + pv * rv.T - rdv.T)
        st["xc"], st["yc"] = x_, y_
        xc.copy_(torch.from_numpy(x_))
        yc.copy_(torch.from_numpy(y_))

    def admm_shard_status(self, st):
        return st["k"], st["done"], st["iters"], st["div"]

    # ---- sharded selection ----
    def to_f64(self, Z, S):
        return Z.clone().double()

    def picked_mask(self, n):
        return torch.zeros(n, dtype=torch.uint8)

    def argmax(self, v, picked, valid=None):
        x = v.numpy().copy()
        p = picked.numpy().astype(bool)
        if valid is None:
            x[p] = 0.0
        else:
            x[p | ~valid.numpy().astype(bool)] = -np.finfo(np.float64).max
        j = int(np.argmax(x))
        return float(x[j]), j

    def spa_step(self, W, s, v, picked):
        w = W[:, :s].numpy()
        if v is not None:
            vv = v[:s].numpy()
            w -= np.outer(w @ vv, vv)
        sq = (w * w).sum(axis=1)
        sq[picked.numpy().astype(bool)] = 0.0
        return torch.from_numpy(sq)

    def col_mass(self, W, s, mass):
        return torch.from_numpy(W[:, :s].numpy() @ mass[:s].numpy())

    def xray_scores(self, W, s, rj, denom):
        return torch.from_numpy((W[:, :s].numpy() @ rj[:s].numpy()) / denom.numpy())

    def right_factor_given(self, W, s, P, k, tol):
        c = P[:k, :s].numpy().T
        h = O.nnls(c, W[:, :s].numpy().T, tol=tol)
        return torch.from_numpy(np.ascontiguousarray(h.T)), 0

    def refit_given(self, W, s, P, k, Ht, R=None):
        w = W[:, :s].numpy()
        res = w - (Ht.numpy() @ P[:k, :s].numpy() if k else 0.0)
        if R is not None:
            R[:, :s] = torch.from_numpy(res)
        sq = (res * res).sum(axis=1)
        return torch.from_numpy(sq), torch.tensor([float(sq.sum()), float((w * w).sum())], dtype=torch.float64)

    def columns_f64(self, A, idx):
        return torch.from_numpy(A.a[:, idx])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _jobs(rank, world, a, a_sep):
    """Every sharded computation the tests check, on this rank's shards."""
    comm, ops = D.Comm(), NumpyOps()
    res = {}
    m, n = a.shape
    c0, ni = D.column_shard(n, world, rank)
    A = Shard(a[:, c0: c0 + ni])
    counts = [D.column_shard(n, world, k)[1] for k in range(world)]
    cfg = adjust_config(CompressionConfig(r=4, r_ov=6, w=2, seed=11), m, n)
    L = D.range_finder(ops, comm, A, m, n, c0, cfg, 0)
    R = comm.allgather_rows(D.range_finder(ops, comm, A, m, n, c0, cfg, 1), counts)
    res["bases"] = (L[:, : cfg.basis_cols].numpy(), R[:, : cfg.basis_cols].numpy())
    # the interleaved pair (forward pass's all-reduce overlapped with the other
    # chain's transpose) against the two sequential finders, same seeds
    from dataclasses import replace
    lcfg = replace(cfg, seed=O.child_seed(11, "left-basis"))
    rcfg = replace(cfg, seed=O.child_seed(11, "right-basis"))
    Li, Ri = D.range_finders_interleaved(ops, comm, A, m, n, c0, lcfg, rcfg)
    Ls = D.range_finder(ops, comm, A, m, n, c0, lcfg, 0)
    Rs = D.range_finder(ops, comm, A, m, n, c0, rcfg, 1)
    res["interleaved"] = (Li.numpy(), Ls.numpy(), comm.allgather_rows(Ri, counts).numpy(),
                          comm.allgather_rows(Rs, counts).numpy())
    u, vt_local, it, _, rel = D.nmf_admm(A, m, n, c0, 4, CompressionConfig(r=4, r_ov=6, w=2, seed=11), comm, ops,
                                         max_iter=60, tol=1e-4)
    res["admm"] = (u.numpy(), comm.allgather_rows(vt_local, counts).numpy(), it, rel)
    m, n = a_sep.shape
    c0, ni = D.column_shard(n, world, rank)
    A = Shard(a_sep[:, c0: c0 + ni])
    cfg = adjust_config(CompressionConfig(r=4, r_ov=6, w=2, seed=11), m, n)
    Q, W = D.reduced_matrix(ops, comm, A, m, n, c0, cfg)
    res["snmf"] = (O.spa(W[:, : cfg.basis_cols].numpy().T, 4), Q[:, : cfg.basis_cols].numpy())
    for sel in ("spa", "xray"):
        out = D.snmf(ops, comm, A, m, n, c0, 4, selector=sel, cfg=CompressionConfig(r=4, r_ov=6, w=2, seed=11),
                     host_out=True)
        res["dsnmf_" + sel] = (out.K, out.Y, out.rel_error_reduced, out.rel_error_full)
    return res


def _worker(rank, world, port, a, a_sep, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _jobs(rank, world, a, a_sep)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def _near_separable():
    return O.near_separable(60, 47, 4, 1.0, 0.001, seed=5)[0]


@pytest.fixture(scope="module")
def mat():
    # uneven shards: n odd
    return O.dense_lowrank(90, 71, 4, 0.01, seed=3)


@pytest.fixture(scope="module")
def sharded(mat):
    """One world-size-2 gloo run computing every sharded result."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mat, _near_separable(), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_column_shard_covers_range():
    for n, w in ((10, 3), (7, 8), (100, 4), (5001, 8)):
        spans = [D.column_shard(n, w, r) for r in range(w)]
        assert spans[0][0] == 0
        assert all(a[0] + a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert spans[-1][0] + spans[-1][1] == n
        assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1


def test_omega_rows_match_full_test_matrix():
    ops = NumpyOps()
    full = O.test_matrix(9000, 5, 17)
    seed = O.child_seed(17, "omega")
    for row0, rows in ((0, 10), (4090, 20), (4096, 4096), (8000, 1000)):
        got = ops.omega_rows(seed, row0, rows, 5, 32)[:, :5].numpy()
        np.testing.assert_array_equal(got, full[row0: row0 + rows])


def test_sharded_bases_match_oracle(mat, sharded):
    L, R = sharded["bases"]
    cfg = O.adjust(O.Config(4, 6, 2, 11), *mat.shape)
    assert O.projector_distance(L, O.range_basis(mat, cfg)) < 1e-10
    assert O.projector_distance(R, O.row_basis(mat, cfg)) < 1e-10
    # identical columns (same canonical signs), not only the same span
    np.testing.assert_allclose(L, O.range_basis(mat, cfg), atol=1e-9)


def test_interleaved_range_finders_equal_sequential(sharded):
    Li, Ls, Ri, Rs = sharded["interleaved"]
    np.testing.assert_array_equal(Li, Ls)
    np.testing.assert_array_equal(Ri, Rs)


def test_sharded_admm_matches_oracle(mat, sharded):
    u, vt, it, rel = sharded["admm"]
    ref = O.admm(mat, 4, cfg=O.Config(4, 6, 2, 11), max_iter=60, tol=1e-4)
    assert it == ref.iterations
    np.testing.assert_allclose(u, ref.X, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(vt.T, ref.Y, rtol=1e-6, atol=1e-9)
    assert abs(rel - ref.rel_error) <= 1e-9 * max(1.0, ref.rel_error)


def test_sharded_reduced_matrix_spa_matches_oracle(sharded):
    a = _near_separable()
    picks, Q = sharded["snmf"]
    ref = O.snmf(a, 4, selector="spa", cfg=O.Config(4, 6, 2, 11))
    np.testing.assert_array_equal(np.sort(picks), np.sort(ref.K))
    np.testing.assert_array_equal(picks, ref.K)


@pytest.mark.parametrize("sel", ["spa", "xray"])
def test_sharded_snmf_matches_oracle(sharded, sel):
    # column-sharded selection: every pick is an all-gather of (score, global
    # index) pairs, the NNLS right factor is column-local
    a = _near_separable()
    K, Y, rr, rf = sharded["dsnmf_" + sel]
    ref = O.snmf(a, 4, selector=sel, cfg=O.Config(4, 6, 2, 11))
    np.testing.assert_array_equal(K, ref.K)
    np.testing.assert_allclose(Y, ref.Y, rtol=1e-7, atol=1e-9)
    assert abs(rr - ref.rel_error_reduced) <= 1e-9
    assert abs(rf - ref.rel_error_full) <= 1e-9


def test_best_pair_tie_rule():
    # (value, global index) all-gather reduction: max value, lowest index
    c = D.Comm()
    assert c.best_pair(3.0, 7) == (3.0, 7)
