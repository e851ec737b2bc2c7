"""Kernel timeline (CUPTI via torch.profiler) of one eager compressed problem
on configs[1]: start/end per kernel and stream, to see the two chains overlap."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem

M, N, R = 10000, 5000, 20
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.rand(M, N, device="cuda", generator=g)
A = DeviceMatrix(a)
cfg = C.adjust_config(C.CompressionConfig(r=R, r_ov=10, w=4, seed=5), M, N)
graph = len(sys.argv) > 1 and sys.argv[1] == "graph"
for _ in range(3):
    compressed_problem(A, cfg, graph=graph)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    compressed_problem(A, cfg, check=False, graph=graph)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    nm = e.name.replace("void cnmf::(anonymous namespace)::", "")[:40]
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:7.1f} "
          f"s{getattr(e, 'device_resource_id', '?')} {nm}")
