"""Per-kernel device times of the streaming ADMM on a configs[4]-sized
compressed problem (m=200000, n=100000, s=60, r=50), via CUPTI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections

import torch
from torch.profiler import ProfilerActivity, profile

import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import zeros
from paper_1505_04650_b200.nmf import run_admm

m, n, r, s = 200_000, 100_000, 50, 60
g = torch.Generator(device="cuda").manual_seed(0)
lp = zeros((m, 64))
rp = zeros((n, 64))
lp[:, :s] = torch.linalg.qr(torch.randn(m, s, device="cuda", generator=g))[0]
rp[:, :s] = torch.linalg.qr(torch.randn(n, s, device="cuda", generator=g))[0]
core = torch.rand(s, s, device="cuda", dtype=torch.float64, generator=g) * 100
cfg = C.CompressionConfig(r=r, r_ov=10, w=4, seed=1)
run_admm(core, lp, m, rp, n, cfg, r, max_iter=3, tol=0.0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run_admm(core, lp, m, rp, n, cfg, r, max_iter=10, tol=0.0)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.replace("(anonymous namespace)", "")[:60]
        agg[k][0] += 1
        agg[k][1] += e.time_range.end - e.time_range.start
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} us {c:5d} launches {t / c:9.1f} us avg  {k}")
