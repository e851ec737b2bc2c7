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
* the ADMM (nmf.py:334-377) acts on O((m + n) r) compressed state and runs
  replicated after one all-gather of R^T; the final ||A - X Y||_F is two
  scalars all-reduced;
* SNMF: the reduced matrix Q^T A (s x n) is gathered once (s * n values, far
  smaller than A) and the column selection runs replicated -- one collective
  instead of an all-reduce of (norm, index) plus a broadcast per pick; the
  picked columns of A are assembled with one all-reduce for the full error.

Collectives go through `Comm` (torch.distributed: NCCL between GPUs, gloo in
the CPU tests); local arithmetic through an ops object -- `DeviceOps` (the C
ABI, the product path) or a test double with the same methods.
"""

from dataclasses import replace

import numpy as np
import torch
import torch.distributed as dist

from .compress import OMEGA_CHUNK, CompressionConfig, adjust_config
from .rng import child_seed


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

    def admm(self, core, left, m, right, n, cfg, r, **kw):
        from .nmf import run_admm

        return run_admm(core, left, m, right, n, cfg, r, **kw)

    def residual(self, A, X, Yt):
        """(||A - X Y||^2, ||A||^2) over the local shard, fp64 device vector."""
        res = self.zeros((2,), torch.float64)
        self._lib.call("cnmf_residual_norms", A.ptr, A.m, A.n, A.lda, X.data_ptr(), None, Yt.data_ptr(),
                       X.shape[1], res.data_ptr(), self._st())
        return res


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


def compressed_problem(ops, comm, A, m, n, c0, cfg):
    """Left basis (replicated), local rows of the right basis, and the core
    L^T A R^T (nmf.py:120-135, 327-332)."""
    left = range_finder(ops, comm, A, m, n, c0, replace(cfg, seed=child_seed(cfg.seed, "left-basis")), 0)
    right = range_finder(ops, comm, A, m, n, c0, replace(cfg, seed=child_seed(cfg.seed, "right-basis")), 1)
    S = left.shape[1]
    core = comm.allreduce(ops.cross(ops.transpose(A, left, S), right, S))
    s = cfg.basis_cols
    return left, right, core[:s, :s].contiguous()


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
    counts = [column_shard(n, comm.world, k)[1] for k in range(comm.world)]
    right = comm.allgather_rows(right_local, counts)
    u, vt, iters, trace = ops.admm(core, left, m, right, n, cfg, r, penalty_u=penalty_u, penalty_v=penalty_v,
                                   step_scale=step_scale, max_iter=max_iter, tol=tol)
    vt_local = vt[c0: c0 + A.n].contiguous()
    res = comm.allreduce(ops.residual(A, u, vt_local))
    num, den = (float(x) for x in res.tolist())
    rel = float(np.sqrt(max(num, 0.0) / den)) if den > 0 else float("nan")
    return u, vt_local, iters, trace, rel


def reduced_matrix(ops, comm, A, m, n, c0, cfg):
    """(Q, W): Q the replicated column basis, W = (Q^T A)^T gathered on every
    rank (n x S) -- the input of the compressed column selection (snmf.py:154-168)."""
    Q = range_finder(ops, comm, A, m, n, c0, cfg, 0)
    S = Q.shape[1]
    counts = [column_shard(n, comm.world, k)[1] for k in range(comm.world)]
    W = comm.allgather_rows(ops.transpose(A, Q, S), counts)
    return Q, W
