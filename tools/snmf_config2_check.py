"""configs[2]-shaped SNMF (tall-skinny, Dirichlet(0.5)) on the SAME numpy
data for the device and the oracle: picks, errors, and whether either raises."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1505_04650_b200 as C
from oracle import cnmf_oracle as O

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
for seed in (1, 2):
    a, truth = O.near_separable(m, 200, 20, 0.5, 0.005, seed=seed)
    a = a.astype(np.float32)
    out = {}
    for name, fn in (("device", lambda: C.snmf(a, 20, selector="spa", cfg=C.CompressionConfig(r=20, r_ov=10, w=2, seed=7))),
                     ("oracle", lambda: O.snmf(a.astype(np.float64), 20, selector="spa", cfg=O.Config(20, 10, 2, 7)))):
        t = time.time()
        try:
            res = fn()
            out[name] = (sorted(np.asarray(res.K).tolist()), float(res.rel_error_full), time.time() - t)
        except Exception as e:
            out[name] = (type(e).__name__, str(e)[:80], time.time() - t)
    same = out["device"][0] == out["oracle"][0]
    print(f"m={m} seed={seed}: device {out['device'][1:]} oracle {out['oracle'][1:]} same picks {same} "
          f"true picked {len(set(out['device'][0]) & set(truth.tolist())) if isinstance(out['device'][0], list) else '-'}",
          flush=True)
