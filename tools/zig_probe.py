"""Time the seeded Gaussian test matrices of configs[4] (rows x 60 in 4096-row
chunks) and print a checksum (compare libraries: the stream must not change)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04650_b200 as C
from torch.profiler import ProfilerActivity, profile
from dataclasses import replace
base = C.CompressionConfig(r=50, r_ov=10, w=4, seed=5)
for rows, side in ((100000, "left-basis"), (200000, "right-basis"), (100000, "right-basis"), (200000, "left-basis")):
    cfg = replace(base, seed=C.child_seed(5, side))
    om = C.draw_test_matrix(cfg, rows)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        om = C.draw_test_matrix(cfg, rows)
        torch.cuda.synchronize()
    ks = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            ks[e.name[:30]] = ks.get(e.name[:30], 0) + (e.time_range.end - e.time_range.start)
    print(rows, side, "sum", float(om.double().sum()), "abs", float(om.double().abs().sum()), {k: round(v) for k, v in ks.items()}, flush=True)
