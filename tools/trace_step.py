"""Timeline of one configs[1] compression (+ short ADMM) via torch.profiler
(CUPTI): per-kernel device time and the idle gaps between kernels."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix
from paper_1505_04650_b200.nmf import compressed_problem

M, N, R = 10000, 5000, 20
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.addmm(0.01 * torch.randn(M, N, device="cuda", generator=g), torch.rand(M, R, device="cuda", generator=g),
                torch.rand(R, N, device="cuda", generator=g)).clamp_(min=0)
A = DeviceMatrix(a)
cfg = C.adjust_config(C.CompressionConfig(r=R, r_ov=10, w=4, seed=5), M, N)
what = sys.argv[1] if len(sys.argv) > 1 else "compress"
def job():
    if what == "compress":
        compressed_problem(A, cfg)
    else:
        C.nmf_admm(A, R, cfg=C.CompressionConfig(r=R, r_ov=10, w=4, seed=5), max_iter=50, tol=0.0)
for _ in range(2):
    job()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    job()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs])
if not ks:
    print("no device events"); sys.exit()
t0, t1 = ks[0][0], max(k[1] for k in ks)
busy = sum(k[1] - k[0] for k in ks)
print(f"span {t1 - t0:.1f} us, device busy {busy:.1f} us, kernels/copies {len(ks)}")
import re
def short(n):
    m = re.findall(r"([A-Za-z_][A-Za-z0-9_]*(?:<[^()]*?>)?)\(", n)
    return (m[0] if m else n)[:50]
agg = {}
for s, e, n in ks:
    key = short(n)
    c, t = agg.get(key, (0, 0.0)); agg[key] = (c + 1, t + e - s)
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{t:9.1f} us  n={c:4d}  avg={t/c:8.2f}  {k}")
gaps = []
for i in range(1, len(ks)):
    gap = ks[i][0] - max(k[1] for k in ks[:i])
    if gap > 15:
        gaps.append((gap, short(ks[i - 1][2]), short(ks[i][2])))
print("largest idle gaps:")
for g_, a_, b_ in sorted(gaps, reverse=True)[:15]:
    print(f"  {g_:8.1f} us  after {a_}  before {b_}")
print(f"total gap {sum(x[0] for x in gaps):.1f} us in {len(gaps)} gaps > 15us")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
cagg = {}
for e in cpu:
    c, t = cagg.get(e.name, (0, 0.0)); cagg[e.name] = (c + 1, t + e.cpu_time_total)
print("host ops (self+children us):")
for k, (c, t) in sorted(cagg.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{t:9.1f}  n={c:4d}  {k[:70]}")
