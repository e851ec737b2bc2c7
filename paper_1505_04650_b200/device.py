"""Device-memory plumbing: moving reference-style inputs onto the GPU in the
layouts the C ABI expects (include/cnmf_b200.h) and handing results back in
the caller's flavour (numpy in -> numpy out, CUDA tensor in -> CUDA tensor out).

torch is used only for allocation, copies and the current stream.
"""

import numpy as np
import torch

from . import _lib
from .errors import ArgumentError, DeviceError

MASK64 = (1 << 64) - 1


def require_cuda():
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the cnmf B200 path runs on the GPU only (no CPU fallback)")
    _lib.load()


def stream():
    return ctypes_stream(torch.cuda.current_stream())


def ctypes_stream(s):
    return s.cuda_stream


def ptr(t):
    return t.data_ptr() if t is not None else None


def panel_ld(s):
    ld = _lib.load().cnmf_panel_ld(int(s))
    if ld < 0:
        raise ArgumentError(f"basis width {s} exceeds the supported maximum of 128")
    return ld


class DeviceMatrix:
    """A (m x n) as fp32 row-major on the device with lda % 4 == 0.

    Numpy / CPU inputs are copied (and padded when n % 4 != 0); a contiguous
    fp32 CUDA tensor with n % 4 == 0 is used in place.
    """

    def __init__(self, a, name="matrix"):
        require_cuda()
        if isinstance(a, DeviceMatrix):
            self.__dict__.update(a.__dict__)
            return
        self.on_host = not (isinstance(a, torch.Tensor) and a.is_cuda)
        if hasattr(a, "to_dense") and not isinstance(a, torch.Tensor):
            a = a.to_dense()  # reference MatrixStore duck type
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if t.dim() != 2:
            raise ArgumentError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
        m, n = t.shape
        if m == 0 or n == 0:
            raise ArgumentError(f"{name} must be non-empty, got shape {tuple(t.shape)}")
        lda = (n + 3) // 4 * 4
        dev = torch.device("cuda", torch.cuda.current_device())
        if (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and lda == n
                and t.data_ptr() % 16 == 0):
            self.t = t
        elif lda == n:
            # one device allocation, one copy (a pinned host matrix is copied
            # asynchronously on the current stream)
            src = t if t.dtype == torch.float32 else t.to(torch.float32)
            buf = torch.empty((m, n), dtype=torch.float32, device=dev)
            buf.copy_(src, non_blocking=src.is_pinned() if not src.is_cuda else True)
            self.t = buf
        else:
            buf = torch.zeros((m, lda), dtype=torch.float32, device=dev)
            buf[:, :n].copy_(t.to(dev, non_blocking=True))
            self.t = buf
        self.m, self.n, self.lda = int(m), int(n), int(lda)

    @property
    def ptr(self):
        return self.t.data_ptr()

    @property
    def shape(self):
        return (self.m, self.n)


class DeviceMatrix64:
    """A (m x n) as fp64 row-major on the device (the fp64 path: float64
    inputs with precision="fp64", BASELINE.json configs[0])."""

    def __init__(self, a, name="matrix"):
        require_cuda()
        if isinstance(a, DeviceMatrix64):
            self.__dict__.update(a.__dict__)
            return
        self.on_host = not (isinstance(a, torch.Tensor) and a.is_cuda)
        if hasattr(a, "to_dense") and not isinstance(a, torch.Tensor):
            a = a.to_dense()
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        if t.dim() != 2:
            raise ArgumentError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
        m, n = t.shape
        if m == 0 or n == 0:
            raise ArgumentError(f"{name} must be non-empty, got shape {tuple(t.shape)}")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.t = t.to(device=dev, dtype=torch.float64).contiguous()
        self.m, self.n, self.lda = int(m), int(n), int(n)

    @property
    def ptr(self):
        return self.t.data_ptr()

    @property
    def shape(self):
        return (self.m, self.n)


def zeros(shape, dtype=torch.float32):
    return torch.zeros(shape, dtype=dtype, device=torch.device("cuda", torch.cuda.current_device()))


def empty(shape, dtype=torch.float32):
    return torch.empty(shape, dtype=dtype, device=torch.device("cuda", torch.cuda.current_device()))


def workspace(nbytes):
    return empty((max(int(nbytes), 16),), dtype=torch.uint8)


def as_device64(x, name):
    """fp64 contiguous device copy of a 2-D array/tensor."""
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    if t.dim() != 2:
        raise ArgumentError(f"{name} must be 2-D")
    return t.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=torch.float64).contiguous()


def out(t, host):
    """Return a device result in the caller's flavour."""
    if host:
        return t.detach().to("cpu").numpy()
    return t


def host_result(shape, dtype=np.float64):
    """A host array for a result that will be copied back later, with its
    pages already touched: meant to be called while the GPU is busy, so the
    page faults of a fresh allocation (most of a pageable D2H's time: 120 MB
    took 56 ms at configs[4]) are off the critical path."""
    buf = np.empty(shape, dtype=dtype)
    buf.fill(0)
    return buf


def out_into(t, buf):
    """Copy a device result into a host array from host_result()."""
    torch.from_numpy(buf).copy_(t.detach())
    return buf


def to_host64(t):
    return t.detach().double().cpu().numpy()
