"""Column-sharded compression, compressed ADMM NMF and compressed SNMF across
the GPUs of one node ("Multi-GPU").

One process per GPU; rank i owns the column shard A[:, c0 : c0 + n_i]
(`column_shard`). The data path touches only the local shard:

* column basis Q (m x s):  Y = sum_i A_i Omega_i  (all-reduce of an m x S
  panel), where rank i draws exactly the Omega rows of its columns (the test
  matrix is generated in 4096-row chunks with one child stream per chunk,
  compress.py:115-127, so any row range is drawable on its own); the
  orthonormalisation of the replicated panel is replicated; a power step is
  Z_i = A_i^T Q (local), Y = sum_i A_i Z_i;
* row basis R^T (n x s): its rows follow the column shards; CholeskyQR of a
  row-sharded panel all-reduces the S x S Gram matrix, factors it on every
  rank and applies R^{-1} locally;
* core L^T A R^T = sum_i (L^T A_i) R_i^T: one S x S all-reduce;
* ADMM (nmf.py:334-377), `admm`: U and dU are row-sharded (rank i updates the
  rows of its row block of L), V^T and dV^T follow the column shards (the rows
  of R_i^T); per iteration every rank sweeps its rows and the s x r reduced
  sums L_i^T U_i, L_i^T dU_i, R_i V_i^T, R_i dV_i^T plus the KKT sums are ONE
  all-reduce of 2 (2 s r + 4) doubles; the core step (KKT score, stopping
  rule, the two r x r ridge solves) runs replicated on identical inputs;
* SNMF (snmf.py:154-232), `snmf`: the reduced matrix stays column-sharded
  ((Q^T A_i)^T on rank i); every SPA / XRAY pick is an all-gather of the
  ranks' (score, global index) pairs -- ties to the lowest index, like
  numpy.argmax -- and the owner of the pick broadcasts the one s-vector
  everybody needs (the normalised column for SPA; the residual column and
  the picked column for XRAY); the NNLS right factor is column-local; the
  full-space error gathers the k picked columns of A once.

Collectives go through `Comm` (torch.distributed: NCCL between GPUs, gloo in
the CPU tests); local arithmetic through an ops object -- `DeviceOps` (the C
ABI, the product path) or a test double with the same methods.
"""

from dataclasses import replace

import numpy as np
import torch
import torch.distributed as dist

from .compress import OMEGA_CHUNK, CompressionConfig, adjust_config
from .errors import ConvergenceError, RankDeficiencyError, UndefinedMetricError
from .rng import child_seed


class _Done:
    def wait(self):
        return True


def column_shard(n, world, rank):
    """Contiguous balanced column range (c0, n_i) of `rank`."""
    base, extra = divmod(int(n), int(world))
    c0 = rank * base + min(rank, extra)
    return c0, base + (1 if rank < extra else 0)


class Comm:
    """The collectives the sharded path needs (SUM all-reduce, row all-gather)."""

    def __init__(self, group=None):
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0

    def allreduce(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def allreduce_async(self, t):
        """Start a SUM all-reduce of `t` in place; the handle's wait() makes
        the caller's stream wait for it (NCCL runs it on its own stream, so a
        kernel enqueued before wait() overlaps the transfer)."""
        if self.world > 1:
            return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        return _Done()

    def allreduce_max(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def best_pair(self, val, idx):
        """Global (max value, lowest index among the maxima) over the ranks'
        local (value, global index) pairs -- numpy.argmax's tie rule."""
        pair = torch.tensor([float(val), float(idx)], dtype=torch.float64, device=self._dev())
        if self.world == 1:
            return float(val), int(idx)
        parts = [torch.empty_like(pair) for _ in range(self.world)]
        dist.all_gather(parts, pair, group=self.group)
        best_v, best_i = None, None
        for p in parts:
            v, i = float(p[0]), int(p[1])
            if best_v is None or v > best_v or (v == best_v and i < best_i):
                best_v, best_i = v, i
        return best_v, best_i

    def _dev(self):
        if dist.is_initialized() and dist.get_backend(self.group) == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def allgather_rows(self, t, counts):
        """Concatenate every rank's (counts[k] x ...) block in rank order."""
        if self.world == 1:
            return t
        mx = max(counts)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]].copy_(t)
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0).contiguous()


class DeviceOps:
    """Local arithmetic through the C ABI (include/cnmf_b200.h)."""

    def __init__(self):
        from . import _lib
        from .device import require_cuda

        require_cuda()
        self._lib = _lib
        self.lib = _lib.load()
        self._status = None

    def begin(self, s):
        """Start a range finder: one small device workspace collects the
        numeric status of every asynchronous step (checked once in end())."""
        nb = int(self.lib.cnmf_small_workspace(s))
        self._status = (torch.empty(nb, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device())),
                        s, nb)
        self._lib.call("cnmf_status_reset", self._status[0].data_ptr(), s, self._st())

    def end(self):
        ws, s, _ = self._status
        self._lib.call("cnmf_status_check", ws.data_ptr(), s, self._st())

    def _st(self):
        from .device import stream

        return stream()

    def panel_ld(self, s):
        from .device import panel_ld

        return panel_ld(s)

    def zeros(self, shape, dtype=torch.float32):
        from .device import zeros

        return zeros(shape, dtype=dtype)

    def omega_rows(self, seed, row0, rows, s, S):
        """Rows [row0, row0 + rows) of the chunked test matrix (compress.py:115)."""
        out = self.zeros((rows, S))
        c_first, c_last = row0 // OMEGA_CHUNK, (row0 + rows - 1) // OMEGA_CHUNK
        for c in range(c_first, c_last + 1):
            start = c * OMEGA_CHUNK
            end = min(row0 + rows, start + OMEGA_CHUNK)
            tmp = self.zeros((end - start, S))  # a chunk's leading rows do not depend on its length
            self._lib.call("cnmf_gaussian_fill", child_seed(seed, f"chunk{c}"), end - start, s, 0, 0,
                           tmp.data_ptr(), S, self._st())
            lo = max(row0, start)
            out[lo - row0: end - row0].copy_(tmp[lo - start:])
        return out

    def forward(self, A, X, S):
        Y = self.zeros((A.m, S))
        self._lib.call("cnmf_pass_forward", A.ptr, A.m, A.n, A.lda, X.data_ptr(), S, Y.data_ptr(), self._st())
        return Y

    def transpose(self, A, W, S):
        Z = self.zeros((A.n, S))
        self._lib.call("cnmf_pass_transpose", A.ptr, A.m, A.n, A.lda, W.data_ptr(), S, Z.data_ptr(), self._st())
        return Z

    def orthonormalize(self, P, s):
        ws, _, nb = self._status
        self._lib.call("cnmf_orthonormalize_async", P.data_ptr(), P.shape[0], s, None, ws.data_ptr(), nb, self._st())
        return P

    def cross(self, P1, P2, S):
        G = self.zeros((S, S), torch.float64)
        self._lib.call("cnmf_panel_cross", P1.data_ptr(), P2.data_ptr(), P1.shape[0], S, G.data_ptr(), self._st())
        return G

    def cholesky_inverse(self, G, s, S):
        T = self.zeros((S, S), torch.float64)
        self._lib.call("cnmf_cholesky_inverse_async", G.data_ptr(), s, S, T.data_ptr(), None,
                       self._status[0].data_ptr(), self._st())
        return T

    def apply(self, P, T, S):
        self._lib.call("cnmf_panel_apply", P.data_ptr(), P.shape[0], S, T.data_ptr(), self._st())
        return P

    def residual(self, A, X, Yt):
        """(||A - X Y||^2, ||A||^2) over the local shard, fp64 device vector."""
        res = self.zeros((2,), torch.float64)
        self._lib.call("cnmf_residual_norms", A.ptr, A.m, A.n, A.lda, X.data_ptr(), None, Yt.data_ptr(),
                       X.shape[1], res.data_ptr(), self._st())
        return res

    # ---- sharded ADMM (include/cnmf_b200.h, "column-sharded multi-GPU") ----
    def uniform(self, seed, start, rows, cols, transpose=False):
        """Rows of the seeded U[0, 1) stream from raw position `start`
        (rng.py:63; nmf.py:337-339's splits, any row block)."""
        t = self.zeros((cols, rows) if transpose else (rows, cols), torch.float64)
        self._lib.call("cnmf_uniform_fill_at", seed, start, rows, cols, 0.0, 1.0, 1, int(bool(transpose)),
                       t.data_ptr(), self._st())
        return t

    def admm_shard_begin(self, s, r, GL, GR):
        nb = int(self.lib.cnmf_admm_shard_workspace(s, r))
        ws = torch.zeros(nb // 8, dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
        self._lib.call("cnmf_admm_shard_begin", ws.data_ptr(), s, r, GL.data_ptr(), GR.data_ptr(), GL.shape[0],
                       self._st())
        off = int(self.lib.cnmf_admm_shard_sums_offset()) // 8
        return {"ws": ws, "sums": ws[off: off + 2 * (2 * s * r + 4)]}

    def admm_shard_sweep(self, st, L, Rt, u, du, vt, dvt, s, r, pu, pv, step, update):
        self._lib.call("cnmf_admm_shard_sweep", st["ws"].data_ptr(), L.data_ptr(), L.shape[0], Rt.data_ptr(),
                       Rt.shape[0], s, r, u.data_ptr(), du.data_ptr(), vt.data_ptr(), dvt.data_ptr(), float(pu),
                       float(pv), float(step), int(update), self._st())
        return st["sums"]

    def admm_shard_core(self, st, core, xc, yc, s, r, pu, pv, step, tol, trace, scores, k, max_iter, first, solve):
        self._lib.call("cnmf_admm_shard_core", st["ws"].data_ptr(), core.data_ptr(), xc.data_ptr(), yc.data_ptr(), s,
                       r, float(pu), float(pv), float(step), float(tol), trace.data_ptr(), scores.data_ptr(), int(k),
                       int(max_iter), int(first), int(solve), self._st())

    def admm_shard_status(self, st):
        import ctypes

        h = (ctypes.c_int * 4)()
        self._lib.call("cnmf_admm_shard_status", st["ws"].data_ptr(), h, self._st())
        return int(h[0]), int(h[1]), int(h[2]), int(h[3])

    # ---- sharded column selection ----
    def to_f64(self, Z, S):
        W = self.zeros((Z.shape[0], S), torch.float64)
        self._lib.call("cnmf_panel_to_f64", Z.data_ptr(), Z.shape[0], S, W.data_ptr(), S, self._st())
        return W

    def picked_mask(self, n):
        return torch.zeros(n, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))

    def argmax(self, v, picked, valid=None):
        out = self.zeros((2,), torch.float64)
        idx = torch.zeros(1, dtype=torch.int64, device=out.device)
        self._lib.call("cnmf_shard_argmax", v.data_ptr(), v.shape[0], picked.data_ptr(),
                       valid.data_ptr() if valid is not None else None, out.data_ptr(), idx.data_ptr(), self._st())
        return float(out[0]), int(idx[0])

    def spa_step(self, W, s, v, picked):
        sq = self.zeros((W.shape[0],), torch.float64)
        self._lib.call("cnmf_spa_shard_step", W.data_ptr(), W.shape[0], s, W.shape[1],
                       v.data_ptr() if v is not None else None, picked.data_ptr(), sq.data_ptr(), self._st())
        return sq

    def col_mass(self, W, s, mass):
        d = self.zeros((W.shape[0],), torch.float64)
        self._lib.call("cnmf_col_mass", W.data_ptr(), W.shape[0], s, W.shape[1], mass.data_ptr(), d.data_ptr(),
                       self._st())
        return d

    def xray_scores(self, W, s, rj, denom):
        sc = self.zeros((W.shape[0],), torch.float64)
        self._lib.call("cnmf_xray_shard_scores", W.data_ptr(), W.shape[0], s, W.shape[1], rj.data_ptr(),
                       denom.data_ptr(), sc.data_ptr(), self._st())
        return sc

    def right_factor_given(self, W, s, P, k, tol):
        import ctypes

        Ht = self.zeros((W.shape[0], k), torch.float64)
        capped = ctypes.c_int64(0)
        self._lib.call("cnmf_right_factor_given", W.data_ptr(), W.shape[0], s, W.shape[1], P.data_ptr(), k,
                       float(tol), Ht.data_ptr(), ctypes.byref(capped), self._st())
        return Ht, int(capped.value)

    def refit_given(self, W, s, P, k, Ht, R=None):
        sq = self.zeros((W.shape[0],), torch.float64)
        tot = self.zeros((2,), torch.float64)
        self._lib.call("cnmf_refit_given", W.data_ptr(), W.shape[0], s, W.shape[1], P.data_ptr(), k,
                       Ht.data_ptr() if Ht is not None else None, R.data_ptr() if R is not None else None,
                       sq.data_ptr(), tot.data_ptr(), self._st())
        return sq, tot

    def columns_f64(self, A, idx):
        """A[:, idx] of the local shard as fp64 (m x len(idx))."""
        if len(idx) == 0:
            return self.zeros((A.m, 0), torch.float64)
        return A.t[:, torch.as_tensor(idx, device=A.t.device)].double()


def orthonormalize_sharded(ops, comm, P, s, S):
    """CholeskyQR2 of a panel whose rows are spread over the ranks."""
    for _ in range(2):
        G = comm.allreduce(ops.cross(P, P, S))
        ops.apply(P, ops.cholesky_inverse(G, s, S), S)
    return P


def range_finder(ops, comm, A, m, n, c0, cfg, side):
    """Distributed structured_compress (side 0, compress.py:156-199: Q, m x S,
    replicated) or structured_compress_rows (side 1, compress.py:202-227: the
    local rows c0 .. c0 + A.n of R^T)."""
    s = cfg.basis_cols
    S = ops.panel_ld(s)
    oseed = child_seed(cfg.seed, "omega")
    ops.begin(s)
    if side == 0:
        Y = comm.allreduce(ops.forward(A, ops.omega_rows(oseed, c0, A.n, s, S), S))
        ops.orthonormalize(Y, s)
        for _ in range(cfg.w):
            Z = orthonormalize_sharded(ops, comm, ops.transpose(A, Y, S), s, S)
            Y = comm.allreduce(ops.forward(A, Z, S))
            ops.orthonormalize(Y, s)
        ops.end()
        return Y
    P = orthonormalize_sharded(ops, comm, ops.transpose(A, ops.omega_rows(oseed, 0, m, s, S), S), s, S)
    for _ in range(cfg.w):
        Y = comm.allreduce(ops.forward(A, P, S))
        ops.orthonormalize(Y, s)
        P = orthonormalize_sharded(ops, comm, ops.transpose(A, Y, S), s, S)
    ops.end()
    return P


def range_finders_interleaved(ops, comm, A, m, n, c0, lcfg, rcfg):
    """Both range finders of nmf_admm, interleaved step by step (the sharded
    counterpart of cnmf_compress_pair_async): at every power step one chain
    needs a forward pass (partial sum, all-reduced) and the other a transpose
    pass (local). The forward pass is enqueued first, its all-reduce is
    started asynchronously, and the transpose pass runs on the GPU while the
    NCCL transfer is in flight; the replicated / sharded orthonormalisations
    follow. Same arithmetic as two range_finder calls (each chain's sequence
    of passes and orthonormalisations is unchanged), so the bases agree
    bit for bit. Returns (Q replicated m x S, this rank's rows of R^T)."""
    if lcfg.w != rcfg.w or lcfg.basis_cols != rcfg.basis_cols:
        return (range_finder(ops, comm, A, m, n, c0, lcfg, 0), range_finder(ops, comm, A, m, n, c0, rcfg, 1))
    s = lcfg.basis_cols
    S = ops.panel_ld(s)
    ops.begin(s)
    # step 0: left Y = sum_i A_i Omega_i (forward), right P = A_i^T Omega' (transpose)
    Y = ops.forward(A, ops.omega_rows(child_seed(lcfg.seed, "omega"), c0, A.n, s, S), S)
    h = comm.allreduce_async(Y)
    P = ops.transpose(A, ops.omega_rows(child_seed(rcfg.seed, "omega"), 0, m, s, S), S)
    h.wait()
    ops.orthonormalize(Y, s)
    P = orthonormalize_sharded(ops, comm, P, s, S)
    for _ in range(lcfg.w):
        # left: Z = A^T Y (transpose), right: Y' = A P (forward, all-reduced)
        Yr = ops.forward(A, P, S)
        h = comm.allreduce_async(Yr)
        Z = ops.transpose(A, Y, S)
        h.wait()
        ops.orthonormalize(Yr, s)
        Z = orthonormalize_sharded(ops, comm, Z, s, S)
        # left: Y = A Z (forward, all-reduced), right: P = A^T Y' (transpose)
        Y = ops.forward(A, Z, S)
        h = comm.allreduce_async(Y)
        P = ops.transpose(A, Yr, S)
        h.wait()
        ops.orthonormalize(Y, s)
        P = orthonormalize_sharded(ops, comm, P, s, S)
    ops.end()
    return Y, P


def compressed_problem(ops, comm, A, m, n, c0, cfg):
    """Left basis (replicated), local rows of the right basis, and the core
    L^T A R^T (nmf.py:120-135, 327-332)."""
    left, right = range_finders_interleaved(ops, comm, A, m, n, c0,
                                            replace(cfg, seed=child_seed(cfg.seed, "left-basis")),
                                            replace(cfg, seed=child_seed(cfg.seed, "right-basis")))
    S = left.shape[1]
    core = comm.allreduce(ops.cross(ops.transpose(A, left, S), right, S))
    s = cfg.basis_cols
    return left, right, core[:s, :s].contiguous()


def admm(ops, comm, core, left, m, right_local, n, c0, cfg, r, penalty_u=1.0, penalty_v=1.0, step_scale=1.0,
         max_iter=500, tol=1e-4, check_every=25):
    """Sharded compressed ADMM (nmf.py:334-377). `left` is the replicated
    left basis (m x S), `right_local` this rank's rows of R^T (n_i x S).
    Rank i updates U rows [m0, m0 + m_i) (`column_shard(m, ...)`) and its
    V^T rows; one all-reduce of the reduced sums per iteration. Returns
    (U m x r assembled on every rank, V^T local rows, iterations, trace)."""
    s = cfg.basis_cols
    m0, mi = column_shard(m, comm.world, comm.rank)
    ni = right_local.shape[0]
    L_loc = left[m0: m0 + mi].contiguous()
    # the seeded U[0, 1) starts (nmf.py:337-339): this rank's U rows are
    # positions [m0 r, (m0 + m_i) r) of the init-left stream; V^T rows of the
    # local columns are taken from the (small) full n x r draw
    u = ops.uniform(child_seed(cfg.seed, "init-left"), m0 * r, mi, r)
    vt = ops.uniform(child_seed(cfg.seed, "init-right"), 0, r, n, transpose=True)[c0: c0 + ni].contiguous()
    du = ops.zeros((mi, r), torch.float64)
    dvt = ops.zeros((ni, r), torch.float64)
    xc = ops.zeros((s, r), torch.float64)
    yc = ops.zeros((r, s), torch.float64)
    trace = ops.zeros((max(max_iter, 1),), torch.float64)
    scores = ops.zeros((max(max_iter, 1),), torch.float64)
    # Gram matrices of the dual-projection recurrence (csrc/admm_stream.cu):
    # G_L = L^T L from the replicated left basis, G_R = sum_i R_i R_i^T
    S = left.shape[1]
    GL = ops.cross(left, left, S)
    GR = comm.allreduce(ops.cross(right_local, right_local, S))
    st = ops.admm_shard_begin(s, r, GL, GR)
    args = (L_loc, right_local, u, du, vt, dvt, s, r, penalty_u, penalty_v, step_scale)
    comm.allreduce(ops.admm_shard_sweep(st, *args, update=0))  # L^T U, V R^T of the start
    for k in range(max_iter):
        ops.admm_shard_core(st, core, xc, yc, s, r, penalty_u, penalty_v, step_scale, tol, trace, scores, k,
                            max_iter, first=(k == 0), solve=1)
        comm.allreduce(ops.admm_shard_sweep(st, *args, update=1))
        if check_every and (k + 1) % check_every == 0 and ops.admm_shard_status(st)[1]:
            break  # every rank takes the same decision (identical all-reduced inputs)
    ops.admm_shard_core(st, core, xc, yc, s, r, penalty_u, penalty_v, step_scale, tol, trace, scores, max_iter,
                        max_iter, first=False, solve=False)
    _, done, iters, diverged = ops.admm_shard_status(st)
    if not done:
        iters = max_iter
    if diverged >= 0:
        from .errors import DivergenceError

        raise DivergenceError(f"KKT residual grew 10x over 50 iterations at iteration {diverged}",
                              trace=scores[: diverged + 1].tolist())
    counts = [column_shard(m, comm.world, k)[1] for k in range(comm.world)]
    u_full = comm.allgather_rows(u, counts)
    return u_full, vt, iters, trace[:iters].tolist()


def rel_error(ops, comm, A, u, vt_local):
    """||A - U V||_F / ||A||_F over the column shards (nmf.py:53-75): two
    scalars all-reduced."""
    res = comm.allreduce(ops.residual(A, u, vt_local))
    num, den = (float(x) for x in res.tolist())
    if den == 0.0:
        raise UndefinedMetricError("relative error undefined: ||A||_F is zero")
    return float(np.sqrt(max(num, 0.0) / den))


def nmf_admm(A, m, n, c0, r, cfg=None, comm=None, ops=None, penalty_u=1.0, penalty_v=1.0, step_scale=1.0,
             max_iter=500, tol=1e-4):
    """Column-sharded compressed ADMM NMF (nmf.py:306-377). `A` is this
    rank's shard (a DeviceMatrix for DeviceOps). Returns (U m x r, V^T rows of
    this shard, iterations, objective trace, relative error)."""
    comm = comm or Comm()
    ops = ops or DeviceOps()
    if cfg is None:
        cfg = CompressionConfig(r=r, r_ov=10, w=4, seed=0)
    cfg = adjust_config(cfg, m, n)
    left, right_local, core = compressed_problem(ops, comm, A, m, n, c0, cfg)
    u, vt_local, iters, trace = admm(ops, comm, core, left, m, right_local, n, c0, cfg, r, penalty_u, penalty_v,
                                     step_scale, max_iter, tol)
    return u, vt_local, iters, trace, rel_error(ops, comm, A, u, vt_local)


def reduced_matrix(ops, comm, A, m, n, c0, cfg):
    """(Q, W): Q the replicated column basis, W = (Q^T A)^T gathered on every
    rank (n x S) -- the input of the compressed column selection (snmf.py:154-168)."""
    Q = range_finder(ops, comm, A, m, n, c0, cfg, 0)
    S = Q.shape[1]
    counts = [column_shard(n, comm.world, k)[1] for k in range(comm.world)]
    W = comm.allgather_rows(ops.transpose(A, Q, S), counts)
    return Q, W


# ------------------------------------------------------------ selection ----

def _owner_row(comm, W, gidx, c0, width):
    """Row `gidx` (global) of the column-sharded W, replicated: the owner
    contributes it, the others zeros, one all-reduce."""
    buf = torch.zeros(width, dtype=W.dtype, device=W.device)
    loc = gidx - c0
    if 0 <= loc < W.shape[0]:
        buf.copy_(W[loc, :width])
    return comm.allreduce(buf)


def select_spa(ops, comm, W, s, r, c0, n):
    """Sharded SPA (snmf.py:39-71) on the local rows of (Q^T A)^T; W is
    projected in place. Picks in order, global column indices."""
    if not 1 <= r <= min(s, n):
        from .errors import ArgumentError

        raise ArgumentError(f"cannot pick {r} columns from a {s}x{n} matrix")
    picked = ops.picked_mask(W.shape[0])
    sq = ops.spa_step(W, s, None, picked)
    smax = comm.allreduce_max(torch.tensor([float(sq.max()) if sq.numel() else 0.0], dtype=torch.float64,
                                           device=comm._dev()))
    floor = (np.sqrt(float(smax[0])) * 1e-14) ** 2
    picks = []
    for _ in range(r):
        v, j = ops.argmax(sq, picked) if sq.numel() else (-1.0, 0)
        v, g = comm.best_pair(v, c0 + j)
        if not v > floor:
            raise RankDeficiencyError(f"only {len(picks)} numerically independent columns found", picks=picks)
        picks.append(g)
        col = _owner_row(comm, W, g, c0, W.shape[1])
        if 0 <= g - c0 < W.shape[0]:
            picked[g - c0] = 1
        vec = (col / np.sqrt(v)).contiguous()
        sq = ops.spa_step(W, s, vec, picked)
    return np.asarray(picks, dtype=np.int64)


def select_xray(ops, comm, W, s, r, c0, n, mass, nnls_tol=1e-10):
    """Sharded XRAY (snmf.py:74-126): per pick, the argmax of the residual
    norms and of the scores are all-gathers of (value, global index); the
    owner broadcasts the residual column and the picked column; the NNLS refit
    of every column is local. Returns (picks, P: the picked columns, k x S)."""
    if not 1 <= r <= min(s, n):
        from .errors import ArgumentError

        raise ArgumentError(f"cannot pick {r} columns from a {s}x{n} matrix")
    S = W.shape[1]
    dev = comm._dev()
    picked = ops.picked_mask(W.shape[0])
    denom = ops.col_mass(W, s, mass)
    dmax = comm.allreduce_max(torch.tensor([float(denom.abs().max()) if denom.numel() else 0.0],
                                           dtype=torch.float64, device=dev))
    scorable = (denom > 1e-14 * max(float(dmax[0]), 1.0)).to(torch.uint8)
    P = torch.zeros((max(r, 1), S), dtype=torch.float64, device=W.device)
    R = W.clone()
    sq, _ = ops.refit_given(W, s, P, 0, None, R)
    smax = comm.allreduce_max(torch.tensor([float(sq.max()) if sq.numel() else 0.0], dtype=torch.float64,
                                           device=dev))
    floor = (np.sqrt(float(smax[0])) * 1e-14) ** 2
    picks = []
    for t in range(r):
        v, j = ops.argmax(sq, picked) if sq.numel() else (-1.0, 0)
        v, gj = comm.best_pair(v, c0 + j)
        if not v > floor:
            raise RankDeficiencyError(f"only {len(picks)} numerically independent columns found", picks=picks)
        rj = _owner_row(comm, R, gj, c0, S)
        score = ops.xray_scores(W, s, rj, denom)
        v, i = ops.argmax(score, picked, scorable) if score.numel() else (-np.inf, 0)
        v, gi = comm.best_pair(v, c0 + i)
        if not (np.isfinite(v) and v > -1.7e308):
            raise RankDeficiencyError("no scorable columns left", picks=picks)
        picks.append(gi)
        P[t].copy_(_owner_row(comm, W, gi, c0, S))
        if 0 <= gi - c0 < W.shape[0]:
            picked[gi - c0] = 1
        Ht, _ = ops.right_factor_given(W, s, P, t + 1, nnls_tol)
        sq, _ = ops.refit_given(W, s, P, t + 1, Ht, R)
    return np.asarray(picks, dtype=np.int64), P[: len(picks)]


def snmf(ops, comm, A, m, n, c0, r, selector="spa", cfg=None, nnls_tol=1e-10, host_out=False):
    """Column-sharded compressed SNMF (snmf.py:154-232): the replicated basis,
    the reduced matrix kept column-sharded, sharded SPA / XRAY, the NNLS right
    factor of the local columns, both relative errors all-reduced. Returns a
    SnmfResult with the picks, Y (all columns, gathered) and the errors."""
    from .snmf import SnmfResult

    if selector not in ("spa", "xray"):
        from .errors import ArgumentError

        raise ArgumentError(f"unknown selector {selector!r}")
    if cfg is None:
        cfg = CompressionConfig(r=r, r_ov=10, w=0, seed=0)
    cfg = adjust_config(cfg, m, n)
    s = cfg.basis_cols
    Q = range_finder(ops, comm, A, m, n, c0, cfg, 0)
    S = Q.shape[1]
    W = ops.to_f64(ops.transpose(A, Q, S), S)  # local rows of (Q^T A)^T
    if selector == "spa":
        picks = select_spa(ops, comm, W.clone(), s, r, c0, n)
        P = torch.stack([_owner_row(comm, W, int(g), c0, S) for g in picks])
    else:
        mass = ops.cross(Q, _ones_panel(ops, Q), S)[:, 0].contiguous()  # Q^T 1 (snmf.py:151, 158)
        picks, P = select_xray(ops, comm, W, s, r, c0, n, mass, nnls_tol)
    k = len(picks)
    Ht, capped = ops.right_factor_given(W, s, P, k, nnls_tol)
    capped_all = comm.allreduce(torch.tensor([float(capped)], dtype=torch.float64, device=comm._dev()))
    counts = [column_shard(n, comm.world, q)[1] for q in range(comm.world)]
    if float(capped_all[0]):
        err = ConvergenceError(f"active-set exchange cap {3 * k} exceeded",
                               best=comm.allgather_rows(Ht, counts).t().cpu().numpy())
        err.picks = picks
        raise err
    _, tot = ops.refit_given(W, s, P, k, Ht, None)
    tot = comm.allreduce(tot)
    res_red, ref_red = (float(x) for x in tot.tolist())
    if ref_red == 0.0:
        raise UndefinedMetricError("reduced matrix has zero norm")
    # full-space error: the picked columns of A, gathered once (m x k)
    own = [int(g) - c0 for g in picks if 0 <= int(g) - c0 < A.n]
    AK = ops.zeros((A.m, k), torch.float64)
    if own:
        cols = ops.columns_f64(A, own)
        pos = [t for t, g in enumerate(picks) if 0 <= int(g) - c0 < A.n]
        AK[:, pos] = cols
    AK = comm.allreduce(AK)
    full = comm.allreduce(ops.residual(A, AK, Ht))
    res_f, ref_f = (float(x) for x in full.tolist())
    Y = comm.allgather_rows(Ht, counts).t().contiguous()
    return SnmfResult(K=np.asarray(picks, dtype=np.int64), Y=Y.cpu().numpy() if host_out else Y,
                      rel_error_reduced=float(np.sqrt(max(res_red, 0.0) / ref_red)),
                      rel_error_full=float(np.sqrt(max(res_f, 0.0) / ref_f)) if ref_f else 0.0)


def _ones_panel(ops, Q):
    o = ops.zeros(tuple(Q.shape), Q.dtype)
    o[:, 0] = 1.0
    return o
