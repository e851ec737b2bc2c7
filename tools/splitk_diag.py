"""Split-K diagnostics for the streaming pass: launch the forward pass many
times on a shape whose output tiles are shared by several CTAs, and for every
corrupted output tile express the error as a combination of the per-CTA
partial sums (which CTA's contribution went missing / was doubled), and which
rows/columns are hit.

usage: python tools/splitk_diag.py m n S reps
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros

m, n, S, reps = (int(v) for v in sys.argv[1:5])
trans = len(sys.argv) > 5 and sys.argv[5] == "t"
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(m + n)
a = torch.rand(m, n, device="cuda", generator=g)
A = DeviceMatrix(a)
K, P = (m, n) if trans else (n, m)
x = torch.randn(K, S, device="cuda", generator=g)
ad = a.double()
yref = (ad.t() if trans else ad) @ x.double()
nt = (K + 31) // 32
nb = (P + 127) // 128
U = nb * nt
G = min(148, U)
bounds = [b * U // G for b in range(G + 1)]
# per (tile, k tile) contributions, fp64: contrib[t, k] = rows of tile t, k tile k
Mt = (ad.t() if trans else ad)
bad_launches = 0
for it in range(reps):
    y = zeros((P, S))
    if trans:
        lib.cnmf_pass_transpose(A.ptr, m, n, A.lda, x.data_ptr(), S, y.data_ptr(), stream())
    else:
        lib.cnmf_pass_forward(A.ptr, m, n, A.lda, x.data_ptr(), S, y.data_ptr(), stream())
    torch.cuda.synchronize()
    err = (y.double() - yref)
    rel = (err.abs().max() / yref.abs().max()).item()
    if rel < 1e-5:
        continue
    bad_launches += 1
    e = err.cpu().numpy()
    rows = np.flatnonzero(np.abs(e).max(axis=1) > 1e-3 * np.abs(yref.cpu().numpy()).max())
    tiles = sorted(set((rows // 128).tolist()))
    print(f"launch {it}: rel {rel:.3e}, {len(rows)} bad rows, tiles {tiles}", flush=True)
    for t in tiles[:4]:
        r0, r1 = t * 128, min(P, t * 128 + 128)
        et = e[r0:r1]
        badr = np.flatnonzero(np.abs(et).max(axis=1) > 1e-3 * np.abs(yref.cpu().numpy()).max())
        badc = np.flatnonzero(np.abs(et).max(axis=0) > 1e-3 * np.abs(yref.cpu().numpy()).max())
        # CTAs touching this tile and their K ranges
        u_t0, u_t1 = t * nt, (t + 1) * nt
        parts = []
        for b in range(G):
            lo, hi = max(bounds[b], u_t0), min(bounds[b + 1], u_t1)
            if lo < hi:
                k0, k1 = lo - u_t0, hi - u_t0
                c = (Mt[r0:r1, 32 * k0:min(K, 32 * k1)] @ x.double()[32 * k0:min(K, 32 * k1)]).cpu().numpy()
                parts.append((b, k0, k1, c))
        # least squares: err = sum_b coef_b * part_b
        Mat = np.stack([p[3].ravel() for p in parts], 1)
        coef, *_ = np.linalg.lstsq(Mat, et.ravel(), rcond=None)
        resid = np.linalg.norm(Mat @ coef - et.ravel()) / max(np.linalg.norm(et), 1e-30)
        desc = ", ".join(f"cta{p[0]}[k{p[1]}:{p[2]}]={c:+.2f}" for p, c in zip(parts, coef) if abs(c) > 0.05)
        print(f"  tile {t}: rows {badr.min()}..{badr.max()} ({len(badr)}), cols {badc.min()}..{badc.max()} "
              f"({len(badc)}); fit resid {resid:.2e}: {desc}", flush=True)
        # per zeroing slice (CTA b zeroes rows [b P / G, (b + 1) P / G)): is the
        # error there a clean combination of CTA partials?
        for zb in range(G):
            z0, z1 = zb * P // G, (zb + 1) * P // G
            lo_, hi_ = max(z0, r0), min(z1, r1)
            if lo_ >= hi_:
                continue
            es = e[lo_:hi_]
            if np.abs(es).max() < 1e-3 * np.abs(yref.cpu().numpy()).max():
                continue
            Ms2 = np.stack([p[3][lo_ - r0:hi_ - r0].ravel() for p in parts], 1)
            c2, *_ = np.linalg.lstsq(Ms2, es.ravel(), rcond=None)
            rs2 = np.linalg.norm(Ms2 @ c2 - es.ravel()) / max(np.linalg.norm(es), 1e-30)
            d2 = ", ".join(f"cta{p[0]}={c:+.2f}" for p, c in zip(parts, c2) if abs(c) > 0.05)
            print(f"    zero-slice cta{zb} rows {lo_}..{hi_ - 1}: resid {rs2:.2e}: {d2}", flush=True)
        # also: is the error a multiple of single k-tile contributions?
        single = []
        for k in range(nt):
            c = (Mt[r0:r1, 32 * k:min(K, 32 * k + 32)] @ x.double()[32 * k:min(K, 32 * k + 32)]).cpu().numpy()
            single.append(c.ravel())
        Ms = np.stack(single, 1)
        cs, *_ = np.linalg.lstsq(Ms, et.ravel(), rcond=None)
        big = [(k, round(float(v), 2)) for k, v in enumerate(cs) if abs(v) > 0.05]
        rs = np.linalg.norm(Ms @ cs - et.ravel()) / max(np.linalg.norm(et), 1e-30)
        print(f"  per-k-tile fit resid {rs:.2e}: {big[:20]}", flush=True)
print(f"{bad_launches}/{reps} launches corrupted")
