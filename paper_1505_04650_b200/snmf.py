"""Separable NMF on the compressed matrix (reference snmf.py, nnls.py).

``snmf(a, r, selector, reduction, cfg, nnls_tol, scratch_dir)`` keeps the
reference signature (snmf.py:170-232): the basis comes from the device range
finder, Q^T A is one transpose pass over A (kept transposed, one reduced
column per row), column selection, the NNLS right factor and both relative
errors run on the device; only the r picked indices and scalars come back
to the host (plus Y when the caller passed host arrays).
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .compress import CompressionConfig, _check, _compress, _compress_f64, _precision, adjust_config
from .device import DeviceMatrix, as_device64, host_result, out, out_into, panel_ld, stream, zeros
from .errors import ArgumentError, ConvergenceError, RankDeficiencyError, UndefinedMetricError


@dataclass
class SnmfResult:
    """Selected column indices (pick order), coefficients, errors (snmf.py:26-32)."""

    K: np.ndarray
    Y: object
    rel_error_reduced: float
    rel_error_full: float


class _Reduced:
    """The reduced matrix R (s x n) held transposed on the device: W[j] = R[:, j]."""

    def __init__(self, W, s, n, host):
        self.W, self.s, self.n, self.host = W, s, n, host
        self.ld = W.shape[1]


def _reduced_from_host(r_mat):
    host = not (isinstance(r_mat, torch.Tensor) and r_mat.is_cuda)
    R = as_device64(r_mat, "reduced matrix")
    s, n = R.shape
    return _Reduced(R.t().contiguous(), s, n, host)


def _spa(red, r):
    if not 1 <= r <= min(red.s, red.n):
        raise ArgumentError(f"cannot pick {r} columns from a {red.s}x{red.n} matrix")
    work = red.W.clone()
    lib = _lib.load()
    nbytes = lib.cnmf_spa_workspace(red.n, red.s)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=work.device)
    picks = (ctypes.c_int64 * r)()
    npk = ctypes.c_int(0)
    status = lib.cnmf_select_spa(work.data_ptr(), red.n, red.s, red.ld, r, picks, ctypes.byref(npk),
                                 ws.data_ptr(), nbytes, stream())
    got = [int(picks[i]) for i in range(npk.value)]
    _lib.check(status, picks=got)
    return np.asarray(got, dtype=np.int64)


def _xray(red, r, mass, nnls_tol):
    if not 1 <= r <= min(red.s, red.n):
        raise ArgumentError(f"cannot pick {r} columns from a {red.s}x{red.n} matrix")
    if mass is None:
        # snmf.py:96-102: all-ones for nonnegative input, else mean direction
        Wt = red.W
        if float(Wt.min()) >= 0:
            mass_t = torch.ones(red.s, dtype=torch.float64, device=Wt.device)
        else:
            norms = torch.linalg.vector_norm(Wt, dim=1)
            keep = norms > 0
            mass_t = (Wt[keep] / norms[keep, None]).sum(dim=0)
    else:
        mass_t = as_device64(np.asarray(mass, dtype=np.float64).reshape(1, -1), "mass").reshape(-1)
    mass_t = mass_t.contiguous()
    picks = (ctypes.c_int64 * r)()
    npk = ctypes.c_int(0)
    status = _lib.load().cnmf_select_xray(red.W.data_ptr(), red.n, red.s, red.ld, r, mass_t.data_ptr(),
                                          float(nnls_tol), picks, ctypes.byref(npk), stream())
    got = [int(picks[i]) for i in range(npk.value)]
    _lib.check(status, picks=got)
    return np.asarray(got, dtype=np.int64)


def select_columns_spa(r_mat, r):
    """Successive projection (snmf.py:39-71); ties break to the lowest index."""
    return _spa(_reduced_from_host(r_mat), r)


def select_columns_xray(r_mat, r, mass=None, nnls_tol=1e-10):
    """XRAY extreme columns with NNLS refits (snmf.py:74-126)."""
    return _xray(_reduced_from_host(r_mat), r, mass, nnls_tol)


def _right_factor(red, picks, nnls_tol):
    """NNLS coefficients of every reduced column over the picked ones; a
    tripped exchange cap raises ConvergenceError (its ``best`` is the capped
    iterate, and ``picks`` the selection it was computed for)."""
    k = len(picks)
    d_picks = torch.as_tensor(np.asarray(picks, dtype=np.int64), device=red.W.device)
    Ht = zeros((red.n, k), dtype=torch.float64)
    capped = ctypes.c_int64(0)
    _lib.call("cnmf_right_factor", red.W.data_ptr(), red.n, red.s, red.ld, d_picks.data_ptr(), k, float(nnls_tol),
              Ht.data_ptr(), ctypes.byref(capped), stream())
    if capped.value:
        err = ConvergenceError(f"active-set exchange cap {3 * k} exceeded", best=Ht.t().cpu().numpy())
        err.picks = np.asarray(picks, dtype=np.int64)
        raise err
    return Ht, d_picks


def snmf_right_factor(r_red, selected, nnls_tol=1e-10):
    """Y >= 0 expressing every column over the selected ones (snmf.py:129-137)."""
    red = _reduced_from_host(r_red)
    sel = np.asarray(selected, dtype=np.int64)
    if sel.size != np.unique(sel).size:
        raise ArgumentError("selected indices must be distinct")
    if sel.size and (sel.min() < 0 or sel.max() >= red.n):
        raise ArgumentError("selected index out of range")
    Ht, _ = _right_factor(red, sel, nnls_tol)
    return out(Ht.t().contiguous(), red.host)


def nnls_solve(c, d, tol=1e-10, max_exchanges=None):
    """min ||d - c h|| s.t. h >= 0 per column (nnls.py:21-111), on the device."""
    vector_target = np.ndim(d) == 1
    host = not (isinstance(c, torch.Tensor) and c.is_cuda)
    C = as_device64(c, "design")
    D = as_device64(d.reshape(-1, 1) if vector_target else d, "targets")
    if tol <= 0:
        raise ArgumentError("tol must be positive")
    if C.shape[0] != D.shape[0]:
        raise ArgumentError(f"design rows {C.shape[0]} != target rows {D.shape[0]}")
    p, q = C.shape
    k = D.shape[1]
    gram = zeros((q, q), dtype=torch.float64)
    target = zeros((k, q), dtype=torch.float64)
    _lib.call("cnmf_gram_f64", C.data_ptr(), p, q, C.data_ptr(), q, gram.data_ptr(), stream())
    _lib.call("cnmf_gram_f64", D.data_ptr(), p, k, C.data_ptr(), q, target.data_ptr(), stream())
    H = zeros((k, q), dtype=torch.float64)
    capped = ctypes.c_int64(0)
    cap = int(max_exchanges) if max_exchanges is not None else 0
    _lib.call("cnmf_nnls_gram", gram.data_ptr(), target.data_ptr(), k, q, float(tol), cap, H.data_ptr(),
              ctypes.byref(capped), stream())
    h = H.t().contiguous()
    if capped.value:
        best = h.cpu().numpy()
        raise ConvergenceError(f"active-set exchange cap {cap or 3 * q} exceeded",
                               best=best[:, 0] if vector_target else best)
    res = out(h, host)
    return res[:, 0] if vector_target else res


def snmf(a, r, selector="spa", reduction="compressed", cfg=None, nnls_tol=1e-10, scratch_dir=None,
         precision="fp32"):
    """Separable NMF A ~ A[:, K] Y (snmf.py:170-232). ``precision="fp64"``
    keeps A and the compression in fp64 (csrc/f64_path.cu; compressed
    reduction only)."""
    if _precision(precision) == "fp64":
        return _snmf_f64(a, r, selector, reduction, cfg, nnls_tol)
    A = DeviceMatrix(a)
    m, n = A.m, A.n
    if not 1 <= r <= min(m, n):
        raise ArgumentError(f"rank {r} out of range for a {m}x{n} matrix")
    if selector not in ("spa", "xray"):
        raise ArgumentError(f"unknown selector {selector!r}")
    yh = None
    if reduction == "compressed":
        if cfg is None:
            cfg = CompressionConfig(r=r, r_ov=10, w=0, seed=0)
        cfg = adjust_config(cfg, m, n)
        if A.on_host:
            # enqueue the range finder, touch the host array of Y while the
            # GPU works (device.host_result), then wait for its status
            basis, _ = _compress(A, cfg, 0, check=False, host_basis=False)
            yh = host_result((r, n))
            _check(basis)
        else:
            basis, _ = _compress(A, cfg, 0, host_basis=False)
        q = basis.panel
    elif reduction == "qr" and n > m:
        # full QR reduction of a fat matrix (snmf.py:140-151): Q is square
        # (m x m) and orthogonal, so Q^T A is a rotation of A. SPA's norms and
        # projections, XRAY's mass functional (Q Q^T 1 = 1) and the NNLS
        # objectives do not depend on which orthogonal Q it is, so Q = I gives
        # the reference's selections and errors without factorising anything
        if m > 128:
            raise ArgumentError("qr reduction of a fat matrix on the device needs m <= 128")
        S = panel_ld(m)
        q = zeros((m, S))
        q[:, :m] = torch.eye(m, dtype=q.dtype, device=q.device)
    elif reduction == "qr":
        # full QR reduction of a tall matrix: orthonormalise A itself (n <= 128)
        S = panel_ld(n)
        q = zeros((m, S))
        q[:, :n] = A.t[:, :n]
        ws = torch.empty(2 * S * S * 8 + 256, dtype=torch.uint8, device=q.device)
        _lib.call("cnmf_orthonormalize", q.data_ptr(), m, n, None, ws.data_ptr(), ws.numel(), stream())
    else:
        raise ArgumentError(f"unknown reduction {reduction!r}")
    s = int(min(q.shape[1], min(m, n) if reduction == "qr" else cfg.basis_cols))
    S = q.shape[1]
    # reduced matrix (Q^T A), kept transposed: one transpose pass over A
    z = zeros((n, S))
    _lib.call("cnmf_pass_transpose", A.ptr, m, n, A.lda, q.data_ptr(), s, z.data_ptr(), stream())
    W = zeros((n, S), dtype=torch.float64)
    _lib.call("cnmf_panel_to_f64", z.data_ptr(), n, S, W.data_ptr(), S, stream())
    red = _Reduced(W, s, n, A.on_host)
    if selector == "spa":
        picks = _spa(red, r)
    else:
        # column-mass functional: sums of Q's columns (snmf.py:151, 158)
        ones = zeros((m, S))
        ones[:, 0] = 1.0
        cm = zeros((S, S), dtype=torch.float64)
        _lib.call("cnmf_panel_cross", q.data_ptr(), ones.data_ptr(), m, S, cm.data_ptr(), stream())
        picks = _xray(red, r, cm[:s, 0].cpu().numpy(), nnls_tol)
    Ht, d_picks = _right_factor(red, picks, nnls_tol)
    norms = zeros((2,), dtype=torch.float64)
    _lib.call("cnmf_refit_norms", W.data_ptr(), n, s, S, d_picks.data_ptr(), len(picks), Ht.data_ptr(),
              norms.data_ptr(), stream())
    res_red, ref_red = norms.tolist()
    if ref_red == 0.0:
        raise UndefinedMetricError("reduced matrix has zero norm")
    full = zeros((2,), dtype=torch.float64)
    _lib.call("cnmf_residual_norms", A.ptr, m, n, A.lda, None, d_picks.data_ptr(), Ht.data_ptr(), len(picks),
              full.data_ptr(), stream())
    res_f, ref_f = full.tolist()
    Y = out_into(Ht.t(), yh) if yh is not None else out(Ht.t().contiguous(), A.on_host)
    return SnmfResult(K=picks, Y=Y, rel_error_reduced=float(np.sqrt(max(res_red, 0.0) / ref_red)),
                      rel_error_full=float(np.sqrt(max(res_f, 0.0) / ref_f)) if ref_f else 0.0)


def _snmf_f64(a, r, selector, reduction, cfg, nnls_tol):
    """snmf() with A, the basis and Q^T A in fp64 (the selection, the NNLS
    right factor and the error norms are fp64 on every path)."""
    if reduction != "compressed":
        raise ArgumentError("precision='fp64' supports the compressed reduction")
    if selector not in ("spa", "xray"):
        raise ArgumentError(f"unknown selector {selector!r}")
    from .device import DeviceMatrix64

    A = DeviceMatrix64(a)
    m, n = A.m, A.n
    if not 1 <= r <= min(m, n):
        raise ArgumentError(f"rank {r} out of range for a {m}x{n} matrix")
    if cfg is None:
        cfg = CompressionConfig(r=r, r_ov=10, w=0, seed=0)
    cfg = adjust_config(cfg, m, n)
    basis, _ = _compress_f64(A, cfg, 0)
    q = basis.panel
    s, S = cfg.basis_cols, q.shape[1]
    W = zeros((n, S), dtype=torch.float64)
    _lib.call("cnmf_pass_transpose_f64", A.ptr, m, n, A.lda, q.data_ptr(), s, W.data_ptr(), stream())
    red = _Reduced(W, s, n, A.on_host)
    if selector == "spa":
        picks = _spa(red, r)
    else:
        mass = q[:, :s].sum(dim=0)  # Q^T 1 (snmf.py:151, 158)
        picks = _xray(red, r, mass.cpu().numpy(), nnls_tol)
    Ht, d_picks = _right_factor(red, picks, nnls_tol)
    norms = zeros((2,), dtype=torch.float64)
    _lib.call("cnmf_refit_norms", W.data_ptr(), n, s, S, d_picks.data_ptr(), len(picks), Ht.data_ptr(),
              norms.data_ptr(), stream())
    res_red, ref_red = norms.tolist()
    if ref_red == 0.0:
        raise UndefinedMetricError("reduced matrix has zero norm")
    full = zeros((2,), dtype=torch.float64)
    _lib.call("cnmf_residual_norms_f64", A.ptr, m, n, A.lda, None, d_picks.data_ptr(), Ht.data_ptr(), len(picks),
              full.data_ptr(), stream())
    res_f, ref_f = full.tolist()
    Y = out(Ht.t().contiguous(), A.on_host)
    return SnmfResult(K=picks, Y=Y, rel_error_reduced=float(np.sqrt(max(res_red, 0.0) / ref_red)),
                      rel_error_full=float(np.sqrt(max(res_f, 0.0) / ref_f)) if ref_f else 0.0)
