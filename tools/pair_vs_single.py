"""Paired range finders vs single-chain ones vs the oracle (projector distances)."""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1505_04650_b200 as C
from oracle import cnmf_oracle as O
from paper_1505_04650_b200.compress import _compress
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem
from paper_1505_04650_b200.rng import child_seed

m, n = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (2000, 1000)))
a = O.dense_lowrank(m, n, 20, 0.01, seed=0).astype(np.float32)
A = DeviceMatrix(torch.from_numpy(a).cuda())
cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), m, n)
s = cfg.basis_cols
ocfg = O.adjust(O.Config(20, 10, 4, 5), m, n)
L, R = O.compressed_bases(a.astype(np.float64), ocfg, True)
lcfg = replace(cfg, seed=child_seed(cfg.seed, "left-basis"))
rcfg = replace(cfg, seed=child_seed(cfg.seed, "right-basis"))
pd = O.projector_distance
for rep in range(2):
    sl = _compress(A, lcfg, 0)[0].panel[:, :s].double().cpu().numpy()
    sr = _compress(A, rcfg, 1)[0].panel[:, :s].double().cpu().numpy()
    pl, pr, core = compressed_problem(A, cfg, graph=False)
    pl = pl.panel[:, :s].double().cpu().numpy()
    pr = pr.panel[:, :s].double().cpu().numpy()
    print(f"rep {rep}: single-vs-oracle L {pd(sl, L):.3e} R {pd(sr, R.T):.3e} | pair-vs-oracle L {pd(pl, L):.3e} "
          f"R {pd(pr, R.T):.3e} | pair-vs-single L {pd(pl, sl):.3e} R {pd(pr, sr):.3e} | bitwise {np.array_equal(pl, sl)} {np.array_equal(pr, sr)}")
