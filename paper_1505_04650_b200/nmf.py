"""Compressed ADMM NMF on the B200 (reference nmf.py:226-377).

``nmf_admm(a, r, compressed=True, cfg, penalty_u, penalty_v, step_scale,
max_iter, tol, scratch_dir, on_iteration)`` keeps the reference signature:
left/right bases from the device range finder (nmf.py:120-135), the core
L^T A R^T from one transpose pass plus a panel cross product (nmf.py:329-332),
seeded U[0,1] splits drawn on the device bit-identically to the reference
(nmf.py:337-339), then the whole iteration on the device (csrc/admm.cu) and
the true relative error from one fused residual pass over A (nmf.py:53-75).
"""

import ctypes
import os
from collections import OrderedDict
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib
from .compress import CompressionConfig, _check, _compress_pair, adjust_config
from .device import MASK64, DeviceMatrix, as_device64, host_result, out, out_into, stream, zeros
from .errors import ArgumentError, DivergenceError, UndefinedMetricError
from .rng import Rng, child_seed


@dataclass
class FactorPair:
    """Nonnegative factors plus run metadata (nmf.py:37-50)."""

    X: object
    Y: object
    iterations: int
    objective_trace: list = field(default_factory=list)
    rel_error: float = None


@dataclass
class KktResidual:
    """Norms of the six first-order conditions (nmf.py:246-270); the max is
    the ADMM's convergence score."""

    grad_left: float
    grad_right: float
    feas_left: float
    feas_right: float
    comp_left: float
    comp_right: float

    @property
    def max_residual(self):
        return max(self.grad_left, self.grad_right, self.feas_left, self.feas_right, self.comp_left,
                   self.comp_right)


def kkt_residual(state, a_comp, left, right):
    """The six KKT norms at an ADMM state (nmf.py:273-303); ``left`` / ``right``
    are the bases (None = identity). A diagnostic: the products run as fp64
    tensor ops on the device (the ADMM kernels evaluate the same score in
    csrc/admm*.cu on every iteration)."""
    def dev(x):
        return None if x is None else as_device64(x, "state")

    xc, yc, u, v, du, dv = (dev(getattr(state, k)) for k in ("xc", "yc", "u", "v", "dual_u", "dual_v"))
    ac, L, R = dev(a_comp), dev(left), dev(right)
    e = xc @ yc - ac
    ltdu = du if L is None else L.t() @ du
    dvrt = dv if R is None else dv @ R.t()
    lxc = xc if L is None else L @ xc
    ycr = yc if R is None else yc @ R
    nrm = torch.linalg.norm
    out_ = KktResidual(
        float(nrm(e @ yc.t() + ltdu)), float(nrm(xc.t() @ e + dvrt)), float(nrm(lxc - u)), float(nrm(ycr - v)),
        float(torch.sqrt(((du * u) ** 2).sum() + (du.clamp(min=0) ** 2).sum() + ((-u).clamp(min=0) ** 2).sum())),
        float(torch.sqrt(((dv * v) ** 2).sum() + (dv.clamp(min=0) ** 2).sum() + ((-v).clamp(min=0) ** 2).sum())))
    return out_


@dataclass
class AdmmState:
    """ADMM iterates (nmf.py:232-244): compressed cores, splits, duals."""

    xc: object
    yc: object
    u: object
    v: object
    dual_u: object
    dual_v: object
    penalty_u: float
    penalty_v: float
    step_scale: float


def _resolve_config(r, cfg, m, n):
    """nmf.py:108-117."""
    if cfg is None:
        cfg = CompressionConfig(r=r, r_ov=10, w=4, seed=0)
    if cfg.r != r:
        raise ArgumentError(f"cfg.r = {cfg.r} disagrees with rank argument {r}")
    return adjust_config(cfg, m, n)


def relative_error(a, x, y):
    """||A - X Y||_F / ||A||_F from one fused pass over A (nmf.py:53-75)."""
    A = DeviceMatrix(a)
    X = as_device64(x, "X")
    Y = as_device64(y, "Y")
    if X.shape[0] != A.m or Y.shape[1] != A.n or X.shape[1] != Y.shape[0]:
        raise ArgumentError(f"shape mismatch: A {A.shape}, X {tuple(X.shape)}, Y {tuple(Y.shape)}")
    return _rel_error(A, X, Y.t().contiguous())


def _rel_error(A, X, Yt):
    res = zeros((2,), dtype=torch.float64)
    _lib.call("cnmf_residual_norms", A.ptr, A.m, A.n, A.lda, X.data_ptr(), None, Yt.data_ptr(), X.shape[1],
              res.data_ptr(), stream())
    num, den = res.tolist()
    if den == 0.0:
        raise UndefinedMetricError("relative error undefined: ||A||_F is zero")
    return float(np.sqrt(max(num, 0.0) / den))


def _enqueue_problem(A, cfg):
    left, right = _compress_pair(A, replace(cfg, seed=child_seed(cfg.seed, "left-basis")),
                                 replace(cfg, seed=child_seed(cfg.seed, "right-basis")))
    s = cfg.basis_cols
    S = left.panel.shape[1]
    z = zeros((A.n, S))
    _lib.call("cnmf_pass_transpose", A.ptr, A.m, A.n, A.lda, left.panel.data_ptr(), s, z.data_ptr(), stream())
    core = zeros((S, S), dtype=torch.float64)
    _lib.call("cnmf_panel_cross", z.data_ptr(), right.panel.data_ptr(), A.n, S, core.data_ptr(), stream())
    return left, right, core, z


# CUDA graphs of the whole compressed problem (2 x (2q+1) passes, their
# CholeskyQR sweeps, the seeded test matrices and the core projection: ~60
# launches) for device-resident A, keyed by everything the launches bake in:
# A's address and shape, the basis width, q and the seed. A replay reuses the graph's own
# output buffers, so the returned bases are valid until the next call with
# the same key. CNMF_GRAPHS=0 runs the launches eagerly.
_GRAPHS = OrderedDict()
_GRAPHS_MAX = 4
graph_launches = 0  # library kernels launched through graph replays (cnmf_launch_count sees captures only)


def _graphs_enabled():
    return os.environ.get("CNMF_GRAPHS", "1") != "0"


def compressed_problem(A, cfg, check=True, graph=None, host_bases=True):
    """Bases and core for the compressed ADMM (nmf.py:120-135, 327-332),
    enqueued back to back (replayed as one CUDA graph unless graph=False or
    CNMF_GRAPHS=0); one status check at the end."""
    # host inputs land in a fresh device buffer per call: a graph keyed on its
    # address would be re-captured every time, so they run eagerly
    use_graph = (_graphs_enabled() and not A.on_host) if graph is None else graph
    if use_graph and not torch.cuda.is_current_stream_capturing():
        key = (A.ptr, A.m, A.n, A.lda, cfg.basis_cols, cfg.w, cfg.seed & MASK64, torch.cuda.current_device())
        ent = _GRAPHS.get(key)
        if ent is None:
            _enqueue_problem(A, cfg)  # initialises the library's one-time launch state
            torch.cuda.current_stream().synchronize()
            lib = _lib.load()
            g = torch.cuda.CUDAGraph()
            n0 = lib.cnmf_launch_count()
            with torch.cuda.graph(g):
                left, right, core, z = _enqueue_problem(A, cfg)
            ent = (g, left, right, core, z, lib.cnmf_launch_count() - n0)
            _GRAPHS[key] = ent
            while len(_GRAPHS) > _GRAPHS_MAX:
                _GRAPHS.popitem(last=False)
        else:
            _GRAPHS.move_to_end(key)
        g, left, right, core, _, nk = ent
        g.replay()
        global graph_launches
        graph_launches += nk
    else:
        left, right, core, _ = _enqueue_problem(A, cfg)
    s = cfg.basis_cols
    if check:
        _check(left)
        _check(right)
    if A.on_host and host_bases:
        # host copies of the bases for callers that asked for them (nmf_admm
        # does not return them: at configs[4] the two copies were 144 MB of
        # pageable D2H, 60 ms of the end-to-end call)
        left.Q = left.panel[:, :s].double().cpu().numpy()
        right.Q = right.panel[:, :s].double().cpu().numpy()
    return left, right, core[:s, :s].contiguous()


def nmf_admm(a, r, compressed=True, cfg=None, penalty_u=1.0, penalty_v=1.0, step_scale=1.0, max_iter=500,
             tol=1e-4, scratch_dir=None, on_iteration=None):
    """NMF through ADMM on U = L Xc, V = Yc R, U, V >= 0 (nmf.py:306-377)."""
    if penalty_u <= 0 or penalty_v <= 0:
        raise ArgumentError("penalties must be positive")
    A = DeviceMatrix(a)
    m, n = A.m, A.n
    if not compressed:
        return _nmf_admm_full(A, r, cfg, penalty_u, penalty_v, step_scale, max_iter, tol, on_iteration)
    cfg = _resolve_config(r, cfg, m, n)
    if A.on_host:
        # enqueue the compression, then allocate and touch the host arrays of
        # the factors while the GPU works, and only then wait for its status
        left, right, core = compressed_problem(A, cfg, check=False, host_bases=False)
        xh, yh = host_result((m, r)), host_result((r, n))
        _check(left)
        _check(right)
    else:
        left, right, core = compressed_problem(A, cfg, host_bases=False)

    def snapshot(k, u, du, vt, dvt, xc, yc):
        st = AdmmState(xc=out(xc.clone(), A.on_host), yc=out(yc.clone(), A.on_host), u=out(u.clone(), A.on_host),
                       v=out(vt.t().contiguous(), A.on_host), dual_u=out(du.clone(), A.on_host),
                       dual_v=out(dvt.t().contiguous(), A.on_host), penalty_u=penalty_u, penalty_v=penalty_v,
                       step_scale=step_scale)
        on_iteration(k, st)

    u, vt, iters, trace = run_admm(core, left.panel, m, right.panel, n, cfg, r, penalty_u, penalty_v, step_scale,
                                   max_iter, tol, snapshot if on_iteration is not None else None)
    rel = _rel_error(A, u, vt)
    if A.on_host:
        return FactorPair(X=out_into(u, xh), Y=out_into(vt.t(), yh), iterations=iters, objective_trace=trace,
                          rel_error=rel)
    return FactorPair(X=u, Y=vt.t().contiguous(), iterations=iters, objective_trace=trace, rel_error=rel)


def _nmf_admm_full(A, r, cfg, penalty_u, penalty_v, step_scale, max_iter, tol, on_iteration):
    """nmf_admm(compressed=False): the same loop with identity bases and
    a_comp = A (nmf.py:326-335), csrc/admm_full.cu."""
    m, n = A.m, A.n
    if cfg is None:
        cfg = CompressionConfig(r=r, r_ov=10, w=4, seed=0)
    if cfg.r != r:
        raise ArgumentError(f"cfg.r = {cfg.r} disagrees with rank argument {r}")
    if not 1 <= r <= min(m, n):  # nmf.py:113-115
        raise ArgumentError(f"rank {r} out of range for {m}x{n}")
    rng = Rng(cfg.seed)
    u = rng.child("init-left").uniform((m, r))
    vt = rng.child("init-right").uniform((r, n), transpose=True)  # V^T, n x r
    du = zeros((m, r), dtype=torch.float64)
    dvt = zeros((n, r), dtype=torch.float64)
    xc = zeros((m, r), dtype=torch.float64)
    yct = zeros((n, r), dtype=torch.float64)
    trace = zeros((max(max_iter, 1),), dtype=torch.float64)
    scores = zeros((max(max_iter, 1),), dtype=torch.float64)
    lib = _lib.load()
    nbytes = lib.cnmf_admm_full_workspace(m, n, r)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=u.device)
    it = ctypes.c_int(0)
    done = ctypes.c_int(0)
    args = lambda resume, limit: (A.ptr, m, n, A.lda, r, u.data_ptr(), du.data_ptr(), vt.data_ptr(), dvt.data_ptr(),
                                  xc.data_ptr(), yct.data_ptr(), float(penalty_u), float(penalty_v), float(step_scale),
                                  int(max_iter), float(tol), trace.data_ptr(), scores.data_ptr(), ctypes.byref(it),
                                  ctypes.byref(done), resume, limit, ws.data_ptr(), nbytes, stream())

    def diverged():
        return dict(trace=scores[:it.value].tolist())

    if on_iteration is None:
        _lib.check(lib.cnmf_admm_full_run(*args(0, 0)), **diverged())
    else:
        resume = 0
        seen = 0
        while True:
            _lib.check(lib.cnmf_admm_full_run(*args(resume, 1)), **diverged())
            resume = 1
            if it.value > seen:
                seen = it.value
                host = A.on_host
                on_iteration(seen - 1, AdmmState(
                    xc=out(xc.clone(), host), yc=out(yct.t().contiguous(), host), u=out(u.clone(), host),
                    v=out(vt.t().contiguous(), host), dual_u=out(du.clone(), host),
                    dual_v=out(dvt.t().contiguous(), host), penalty_u=penalty_u, penalty_v=penalty_v,
                    step_scale=step_scale))
            if done.value:
                break
    iters = it.value
    rel = _rel_error(A, u, vt)
    return FactorPair(X=out(u, A.on_host), Y=out(vt.t().contiguous(), A.on_host), iterations=iters,
                      objective_trace=trace[:iters].tolist(), rel_error=rel)


def run_admm(core, left_panel, m, right_panel, n, cfg, r, penalty_u=1.0, penalty_v=1.0, step_scale=1.0,
             max_iter=500, tol=1e-4, on_iteration=None):
    """The ADMM loop of nmf.py:334-377 on the device for a compressed problem
    (core = L^T A R^T, s x s fp64; left panel m x S, right panel R^T n x S):
    seeded U[0,1] starts (nmf.py:337-339), then cnmf_admm_run. Returns
    (U m x r, V^T n x r, iterations, objective trace)."""
    s = cfg.basis_cols
    rng = Rng(cfg.seed)
    u = rng.child("init-left").uniform((m, r))
    vt = rng.child("init-right").uniform((r, n), transpose=True)  # V^T, n x r
    du = zeros((m, r), dtype=torch.float64)
    dvt = zeros((n, r), dtype=torch.float64)
    xc = zeros((s, r), dtype=torch.float64)
    yc = zeros((r, s), dtype=torch.float64)
    trace = zeros((max(max_iter, 1),), dtype=torch.float64)
    scores = zeros((max(max_iter, 1),), dtype=torch.float64)
    lib = _lib.load()
    nbytes = lib.cnmf_admm_workspace(m, n, s, r)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=u.device)
    it = ctypes.c_int(0)
    done = ctypes.c_int(0)
    args = lambda resume, limit: (core.data_ptr(), left_panel.data_ptr(), m, right_panel.data_ptr(), n, s, r,
                                  u.data_ptr(), du.data_ptr(), vt.data_ptr(), dvt.data_ptr(), xc.data_ptr(),
                                  yc.data_ptr(), float(penalty_u), float(penalty_v), float(step_scale),
                                  int(max_iter), float(tol), trace.data_ptr(), scores.data_ptr(), ctypes.byref(it),
                                  ctypes.byref(done), resume, limit, ws.data_ptr(), nbytes, stream())

    def diverged():
        return dict(trace=scores[:it.value].tolist())

    if on_iteration is None:
        status = lib.cnmf_admm_run(*args(0, 0))
        _lib.check(status, **diverged())
    else:
        resume = 0
        seen = 0
        while True:
            status = lib.cnmf_admm_run(*args(resume, 1))
            _lib.check(status, **diverged())
            resume = 1
            if it.value > seen:
                seen = it.value
                on_iteration(seen - 1, u, du, vt, dvt, xc, yc)
            if done.value:
                break
    iters = it.value
    return u, vt, iters, trace[:iters].tolist()
