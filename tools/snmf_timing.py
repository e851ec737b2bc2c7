"""Wall time of the device SNMF pipeline vs the oracle on a configs[3]-like problem."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch

import cnmf_oracle as O
import paper_1505_04650_b200 as C

m, n, r = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1200, 1500, 40)))
a, truth = O.near_separable(m, n, r, 1.0, 0.01, seed=31)
a32 = a.astype(np.float32)
for sel in ("spa", "xray"):
    C.snmf(a32, r, selector=sel, cfg=C.CompressionConfig(r=r, r_ov=10, w=4, seed=6))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = C.snmf(a32, r, selector=sel, cfg=C.CompressionConfig(r=r, r_ov=10, w=4, seed=6))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ref = O.snmf(a32.astype(np.float64), r, selector=sel, cfg=O.Config(r, 10, 4, 6))
    t2 = time.perf_counter()
    print(f"{sel}: device {1e3 * (t1 - t0):.1f} ms, oracle {1e3 * (t2 - t1):.1f} ms, same picks {np.array_equal(res.K, ref.K)}")
