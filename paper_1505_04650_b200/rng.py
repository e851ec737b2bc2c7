"""Seeded randomness, drawn on the device (reference rng.py).

The reference wraps numpy's Generator(Philox4x64) with ziggurat normals
(rng.py:38-98). The device sampler (csrc/rng.cu) reproduces those streams
bit for bit, so ``Rng(seed).standard_normal`` here returns exactly the values
the reference would, only as a CUDA tensor. Child seeds are derived on the
host with the reference's FNV-1a/SplitMix64 rule (rng.py:23-35, 56-58, 73-75).
"""

import torch

from . import _lib
from .device import MASK64, empty, require_cuda, stream
from .errors import ArgumentError

ALGORITHM = "philox4x64/ziggurat"


def _fnv1a64(text):
    h = 0xCBF29CE484222325
    for byte in text.encode("utf-8"):
        h = ((h ^ byte) * 0x100000001B3) & MASK64
    return h


def _splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def child_seed(seed, tag):
    """Child seed as a plain integer (rng.py:73-75)."""
    return _splitmix64((int(seed) & MASK64) ^ _fnv1a64(tag))


class Rng:
    """Seeded device stream (rng.py:38-70). Successive draws continue the
    stream like the reference's numpy Generator: the instance tracks the raw
    64-bit draw position (uniform: one raw draw per variate; standard_normal:
    the ziggurat's variable count, reported back by the device sampler).

    ``integers`` and ``permutation`` (rng.py:66-70) draw through numpy's
    bounded-integer samplers (32-bit buffered draws, rejection loops); they are
    not on the compression / NMF / SNMF path and have no device sampler here:
    they raise ``ArgumentError`` ("Rng")."""

    algorithm = ALGORITHM

    def __init__(self, seed):
        self.seed = int(seed) & MASK64
        self._pos = 0  # raw 64-bit draws consumed so far

    def __repr__(self):
        return f"Rng(seed={self.seed}, algorithm={self.algorithm!r})"

    def child(self, tag):
        return Rng(child_seed(self.seed, tag))

    def standard_normal(self, shape, dtype=torch.float64):
        rows, cols = _shape2(shape)
        require_cuda()
        t = empty((rows, cols), dtype=dtype)
        end = torch.zeros(1, dtype=torch.int64, device=t.device)
        _lib.call("cnmf_normal_fill_at", self.seed, self._pos, rows * cols, _code(dtype), t.data_ptr(),
                  end.data_ptr(), stream())
        self._pos = int(end.item())
        return t.reshape(shape)

    def uniform(self, shape, low=0.0, high=1.0, dtype=torch.float64, transpose=False):
        rows, cols = _shape2(shape)
        require_cuda()
        t = empty((cols, rows) if transpose else (rows, cols), dtype=dtype)
        _lib.call("cnmf_uniform_fill_at", self.seed, self._pos, rows, cols, float(low), float(high), _code(dtype),
                  int(bool(transpose)), t.data_ptr(), stream())
        self._pos += rows * cols
        return t if transpose else t.reshape(shape)

    def integers(self, low, high, size=None):
        raise ArgumentError("Rng.integers has no device sampler (not on the compressed-NMF path); "
                            "draw indices with numpy from Rng.child(tag).seed")

    def permutation(self, n):
        raise ArgumentError("Rng.permutation has no device sampler (not on the compressed-NMF path); "
                            "draw permutations with numpy from Rng.child(tag).seed")


def _shape2(shape):
    if isinstance(shape, int):
        return 1, int(shape)
    if len(shape) == 1:
        return 1, int(shape[0])
    if len(shape) != 2:
        raise ArgumentError("only 1-D and 2-D draws are supported")
    return int(shape[0]), int(shape[1])


def _code(dtype):
    if dtype == torch.float64:
        return 1
    if dtype == torch.float32:
        return 0
    raise ArgumentError(f"unsupported dtype {dtype}")


def gaussian_matrix(rows, cols, rng):
    """i.i.d. standard normals, deterministic in the seed (rng.py:78-98)."""
    if rows < 1 or cols < 1:
        raise ArgumentError(f"gaussian_matrix needs positive dims, got {rows}x{cols}")
    if not isinstance(rng, Rng):
        rng = Rng(rng)
    return rng.standard_normal((rows, cols))
