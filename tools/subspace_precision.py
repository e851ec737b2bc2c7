"""Projector distance of the device range finder to the reference's basis at
configs[1] shapes (fixture tests/golden/reference_large.npz), plus the pass
error vs fp64 -- for A/B of pass-kernel precision variants (CNMF_LIB_PATH)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np
import torch

import paper_1505_04650_b200 as C
from make_golden_large import dense_config1, proj_dist

fx = np.load(os.path.join(ROOT, "tests", "golden", "reference_large.npz"))
out = []
for m, n in ((2000, 1000), (10000, 5000)):
    a = dense_config1(m, n, seed=11).astype(np.float32)
    q = C.structured_compress(a, C.CompressionConfig(r=20, r_ov=10, w=4, seed=3)).Q
    key = f"c1_{m}x{n}"
    out.append(f"{key} dist {proj_dist(fx[key + '_q'].astype(np.float64), q):.3e} band {fx[key + '_band'].max():.3e}")
# forward pass error vs fp64 at K = 100000 (configs[4]'s forward K)
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.rand(4096, 100000, device="cuda", generator=g)
x = torch.zeros(100000, 64, device="cuda")
x[:, :60] = torch.randn(100000, 60, device="cuda", generator=g)
from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros
A = DeviceMatrix(a)
y = zeros((4096, 64))
_lib.call("cnmf_pass_forward", A.ptr, 4096, 100000, A.lda, x.data_ptr(), 60, y.data_ptr(), stream())
ref = a.double() @ x.double()
scale = a.double().abs() @ x.double().abs()
e = (y.double() - ref) / scale
out.append(f"K=100000 fwd rel err rms {e.pow(2).mean().sqrt().item():.2e} max {e.abs().max().item():.2e} "
           f"mean {e.mean().item():+.2e}")
print(" | ".join(out), flush=True)
