"""The device's log1p (csrc/glibc_log1p.cuh, used for numpy's ziggurat tail)
compiled for the host and compared bit for bit with the C library's log1p
(what numpy calls) on this machine."""
import math
import os
import shutil
import struct
import subprocess
import tempfile

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
HDR = os.path.join(HERE, "..", "paper_1505_04650_b200", "csrc", "glibc_log1p.cuh")

SRC = r"""
#include "%s"
#include <cstdio>
int main() {
  double x;
  while (fread(&x, 8, 1, stdin) == 1) { double y = cnmf::glibc_log1p(x); fwrite(&y, 8, 1, stdout); }
}
"""


@pytest.fixture(scope="module")
def exe():
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    d = tempfile.mkdtemp()
    src = os.path.join(d, "l1p.cpp")
    with open(src, "w") as f:
        f.write(SRC % os.path.abspath(HDR))
    out = os.path.join(d, "l1p")
    subprocess.run(["g++", "-O2", "-std=c++17", src, "-o", out], check=True)
    return out


def test_log1p_matches_libm(exe):
    g = np.random.default_rng(0)
    u = (g.integers(0, 2**53, size=400_000, dtype=np.uint64).astype(np.float64)) * 2.0**-53
    xs = np.concatenate([-u,                                   # numpy's tail: log1p(-u), u = k 2^-53
                         u * 4 - 1.0, u * 1e6, np.ldexp(u, -40), -np.ldexp(u, -30),
                         [0.0, -0.0, 2.0**-60, -2.0**-29, 0.41421, -0.2929, 1e300]])
    got = np.frombuffer(subprocess.run([exe], input=xs.astype("<f8").tobytes(), capture_output=True,
                                       check=True).stdout, dtype="<f8")
    want = np.array([math.log1p(x) for x in xs])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
