"""Structured random compression on the B200 (reference compress.py).

Public functions keep the reference's signatures:

* ``structured_compress(a, cfg, reorthogonalize=False, scratch_dir=None)``
  (compress.py:156-199) — column-space basis, one C-ABI call
  (``cnmf_structured_compress``) that draws the reference's Gaussian test
  matrix on the device, streams the 2w+1 passes over A and orthonormalises.
* ``structured_compress_rows`` (compress.py:202-227) — row-space basis.
* ``gaussian_compress`` (compress.py:238-247), ``compression_error``
  (compress.py:250-265), ``adjust_config`` (compress.py:101-112),
  ``draw_test_matrix`` (compress.py:125-127).

``reorthogonalize`` is accepted for signature compatibility; the device path
always re-orthonormalises between passes (deferred CholeskyQR, see
csrc/linalg.cu), which yields the same Q as the reference in exact arithmetic
and is the numerically stable variant in floating point.
"""

from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .device import MASK64, DeviceMatrix, DeviceMatrix64, as_device64, empty, out, panel_ld, stream, workspace, zeros
from .errors import ArgumentError, InfeasibleRankError
from .rng import child_seed

OMEGA_CHUNK = 4096  # compress.py:22


@dataclass(frozen=True)
class CompressionConfig:
    """Target rank, oversampling, power passes, seed (compress.py:27-51)."""

    r: int
    r_ov: int = 10
    w: int = 4
    seed: int = 0

    def __post_init__(self):
        if self.r < 1:
            raise ArgumentError(f"target rank must be >= 1, got {self.r}")
        if self.r_ov < 0:
            raise ArgumentError(f"oversampling must be >= 0, got {self.r_ov}")
        if self.w < 0:
            raise ArgumentError(f"power exponent must be >= 0, got {self.w}")

    @property
    def basis_cols(self):
        return self.r + self.r_ov


@dataclass
class CompressionBasis:
    """Basis produced by a compression run (compress.py:54-80).

    ``Q`` is an ndarray (host input) or a CUDA tensor view (device input);
    ``panel`` is the padded device panel the other device kernels consume.
    """

    Q: object
    kind: str
    config: CompressionConfig
    panel: object = None

    @property
    def cols(self):
        return self.Q.shape[1]

    @property
    def rows(self):
        return self.Q.shape[0]

    def q_dense(self):
        return self.Q


def adjust_config(cfg, m, n):
    """min(max(20, r + r_ov), n, m) sizing rule (compress.py:101-112)."""
    if cfg.r >= min(m, n):
        raise InfeasibleRankError(f"rank {cfg.r} infeasible for a {m}x{n} matrix (need r < min(m, n))")
    width = min(max(20, cfg.r + cfg.r_ov), n, m)
    return replace(cfg, r_ov=width - cfg.r)


def _require_feasible(cfg, m, n):
    s = cfg.basis_cols
    if s > min(m, n):
        raise InfeasibleRankError(f"basis width {s} exceeds min(m, n) = {min(m, n)}; adjust_config first")


def _compress(a, cfg, side, check=True, host_basis=True):
    """Device range finder. check=False enqueues without synchronising; the
    caller must then call ``basis.check()`` before trusting the result.
    host_basis=False keeps Q on the device even for a host input (callers
    that only use the panel, e.g. snmf)."""
    A = DeviceMatrix(a)
    _require_feasible(cfg, A.m, A.n)
    s = cfg.basis_cols
    S = panel_ld(s)
    rows = A.m if side == 0 else A.n
    q = empty((rows, S))
    lib = _lib.load()
    nbytes = lib.cnmf_compress_workspace(A.m, A.n, s)
    ws = workspace(nbytes)
    name = "cnmf_structured_compress" if check else "cnmf_structured_compress_async"
    _lib.call(name, A.ptr, A.m, A.n, A.lda, s, cfg.w, cfg.seed & MASK64, side, q.data_ptr(), ws.data_ptr(), nbytes,
              stream())
    view = q[:, :s]
    Q = view.double().cpu().numpy() if (A.on_host and check and host_basis) else view
    basis = CompressionBasis(Q=Q, kind="structured", config=cfg, panel=q)
    basis._ws = ws
    basis._dims = (A.m, A.n, s)
    return basis, A


def _compress_pair(A, cfg_left, cfg_right):
    """Both range finders of the compressed NMF (nmf.py:120-135) in one
    asynchronous C call: the column chain on the current stream, the row chain
    on a side stream joined back into it, each chain's CholeskyQR sweeps
    overlapping the other chain's passes. Call ``_check`` on both bases."""
    if cfg_left.basis_cols != cfg_right.basis_cols or cfg_left.w != cfg_right.w:
        raise ArgumentError("paired range finders need the same width and power exponent")
    _require_feasible(cfg_left, A.m, A.n)
    s = cfg_left.basis_cols
    S = panel_ld(s)
    ql = empty((A.m, S))
    qr = empty((A.n, S))
    lib = _lib.load()
    nbytes = lib.cnmf_compress_workspace(A.m, A.n, s)
    wl = workspace(nbytes)
    wr = workspace(nbytes)
    _lib.call("cnmf_compress_pair_async", A.ptr, A.m, A.n, A.lda, s, cfg_left.w, cfg_left.seed & MASK64,
              cfg_right.seed & MASK64, ql.data_ptr(), qr.data_ptr(), wl.data_ptr(), wr.data_ptr(), nbytes, stream())
    out_ = []
    for q, ws, cfg in ((ql, wl, cfg_left), (qr, wr, cfg_right)):
        basis = CompressionBasis(Q=q[:, :s], kind="structured", config=cfg, panel=q)
        basis._ws = ws
        basis._dims = (A.m, A.n, s)
        out_.append(basis)
    return out_[0], out_[1]


def _check(basis):
    m, n, s = basis._dims
    _lib.call("cnmf_compress_check", basis._ws.data_ptr(), m, n, s, stream())


def _compress_f64(a, cfg, side):
    """The fp64 range finder (csrc/f64_path.cu): A, panels and products in
    fp64, CholeskyQR2 after every pass."""
    A = DeviceMatrix64(a)
    _require_feasible(cfg, A.m, A.n)
    s = cfg.basis_cols
    S = panel_ld(s)
    if S > 64:
        raise ArgumentError("the fp64 range finder supports basis widths <= 64")
    rows = A.m if side == 0 else A.n
    q = zeros((rows, S), dtype=torch.float64)
    nb = _lib.load().cnmf_compress_f64_workspace(A.m, A.n, s)
    ws = workspace(nb)
    _lib.call("cnmf_structured_compress_f64", A.ptr, A.m, A.n, A.lda, s, cfg.w, cfg.seed & MASK64, side,
              q.data_ptr(), ws.data_ptr(), nb, stream())
    view = q[:, :s]
    basis = CompressionBasis(Q=view.cpu().numpy() if A.on_host else view, kind="structured", config=cfg, panel=q)
    basis.precision = "fp64"
    return basis, A


def _precision(p):
    if p not in ("fp32", "fp64"):
        raise ArgumentError(f"precision must be 'fp32' or 'fp64', got {p!r}")
    return p


def structured_compress(a, cfg, reorthogonalize=False, scratch_dir=None, precision="fp32"):
    """Orthonormal basis for the dominant column space of ``a`` (compress.py:156).
    ``precision="fp64"`` selects the fp64 range finder (float64 workloads such
    as BASELINE.json configs[0]); the default streams A in fp32 through the
    3xTF32 tensor-core passes."""
    if _precision(precision) == "fp64":
        return _compress_f64(a, cfg, 0)[0]
    return _compress(a, cfg, 0)[0]


def structured_compress_rows(a, cfg, reorthogonalize=False, scratch_dir=None, precision="fp32"):
    """Orthonormal basis for the dominant row space of ``a`` (compress.py:202)."""
    if _precision(precision) == "fp64":
        return _compress_f64(a, cfg, 1)[0]
    return _compress(a, cfg, 1)[0]


def draw_test_matrix(cfg, rows, dtype=torch.float64):
    """The seeded Gaussian test matrix, bit-identical to the reference's
    (compress.py:125-127), generated on the device."""
    t = empty((rows, cfg.basis_cols), dtype=dtype)
    _lib.call("cnmf_gaussian_fill", child_seed(cfg.seed, "omega"), rows, cfg.basis_cols, OMEGA_CHUNK,
              0 if dtype == torch.float32 else 1, t.data_ptr(), cfg.basis_cols, stream())
    return t


def gaussian_compress(m, s, seed):
    """Q = s^(-1/2) * (m x s Gaussian) (compress.py:238-247), drawn on the device."""
    if s < 1:
        raise ArgumentError(f"projection width must be >= 1, got {s}")
    from .rng import gaussian_matrix

    g = gaussian_matrix(m, s, child_seed(seed, "gaussian-projection"))
    cfg = CompressionConfig(r=s, r_ov=0, w=0, seed=seed)
    return CompressionBasis(Q=(g / np.sqrt(s)).cpu().numpy(), kind="gaussian", config=cfg)


POWER_NORM_SEED = 0x5EC7AA1  # compress.py:23


def compression_error(a, basis, norm="frobenius"):
    """||A - Q Q^T A|| (compress.py:250-265): Frobenius from one transpose
    pass and one fused residual pass over A; spectral by the reference's power
    iteration on the residual (compress.py:268-286: at most 100 steps,
    relative tolerance 1e-6, start vector Rng(0x5EC7AA1).standard_normal(n)),
    with E v = A v - Q (Z^T v) and E^T u = A^T u - Z (Q^T u), Z = A^T Q, so
    every step is one forward and one transpose pass of the device kernels."""
    if norm not in ("frobenius", "spectral"):
        raise ArgumentError(f"unknown norm {norm!r}")
    A = DeviceMatrix(a)
    qd = as_device64(basis.Q if not isinstance(basis.Q, torch.Tensor) else basis.Q, "Q")
    if qd.shape[0] != A.m:
        raise ArgumentError(f"basis rows {qd.shape[0]} != matrix rows {A.m}")
    s = qd.shape[1]
    S = panel_ld(s)
    qp = zeros((A.m, S))
    qp[:, :s] = qd.float()
    z = zeros((A.n, S))
    _lib.call("cnmf_pass_transpose", A.ptr, A.m, A.n, A.lda, qp.data_ptr(), s, z.data_ptr(), stream())
    if norm == "spectral":
        return _spectral_residual_norm(A, qd, z[:, :s].double())
    zt = z[:, :s].double().contiguous()
    res = zeros((2,), dtype=torch.float64)
    _lib.call("cnmf_residual_norms", A.ptr, A.m, A.n, A.lda, qd.data_ptr(), None, zt.data_ptr(), s,
              res.data_ptr(), stream())
    return float(np.sqrt(max(res[0].item(), 0.0)))


def _spectral_residual_norm(A, q, z, max_iter=100, tol=1e-6):
    """compress.py:268-286 on the device (q: m x s, z = A^T q: n x s, fp64)."""
    from .rng import Rng

    v = Rng(POWER_NORM_SEED).standard_normal((1, A.n))[0]
    v = v / torch.linalg.vector_norm(v)
    vp = zeros((A.n, 32))
    up = zeros((A.m, 32))
    av = zeros((A.m, 32))
    atu = zeros((A.n, 32))
    sigma = 0.0
    for _ in range(max_iter):
        vp[:, 0] = v.float()
        _lib.call("cnmf_pass_forward", A.ptr, A.m, A.n, A.lda, vp.data_ptr(), 1, av.data_ptr(), stream())
        u = av[:, 0].double() - q @ (z.t() @ v)
        new_sigma = float(torch.linalg.vector_norm(u))
        if new_sigma == 0.0:
            return 0.0
        u = u / new_sigma
        up[:, 0] = u.float()
        _lib.call("cnmf_pass_transpose", A.ptr, A.m, A.n, A.lda, up.data_ptr(), 1, atu.data_ptr(), stream())
        w = atu[:, 0].double() - z @ (q.t() @ u)
        wnorm = float(torch.linalg.vector_norm(w))
        if wnorm == 0.0:
            return new_sigma
        v = w / wnorm
        if abs(new_sigma - sigma) <= tol * new_sigma:
            return new_sigma
        sigma = new_sigma
    return sigma


def canonical_qr(b):
    """Reduced QR with diag(R) >= 0 (compress.py:136-145) of a tall matrix
    (rows >= columns <= 128), on the device: CholeskyQR2 of the fp32 panel
    (csrc/linalg.cu; every transform upper triangular with a positive
    diagonal, so Q is the sign-canonical factor) and R = Q^T B in fp64."""
    host = not (isinstance(b, torch.Tensor) and b.is_cuda)
    B = as_device64(b, "b")
    m, k = B.shape
    if k > m:
        raise ArgumentError(f"canonical_qr needs rows >= columns, got {m}x{k}")
    S = panel_ld(k)
    P = zeros((m, S))
    P[:, :k] = B.float()
    nb = 2 * S * S * 8 + 256
    ws = workspace(nb)
    _lib.call("cnmf_orthonormalize", P.data_ptr(), m, k, None, ws.data_ptr(), nb, stream())
    Bp = zeros((m, S))
    Bp[:, :k] = B.float()
    Rm = zeros((S, S), dtype=torch.float64)
    _lib.call("cnmf_panel_cross", P.data_ptr(), Bp.data_ptr(), m, S, Rm.data_ptr(), stream())
    R = torch.triu(Rm[:k, :k]).contiguous()
    Q = P[:, :k].double().contiguous()
    return out(Q, host), out(R, host)
