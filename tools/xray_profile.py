"""XRAY on a configs[3]-shaped reduced matrix (s = 60, n = 200000, r = 50:
near-separable, H = [I | Dirichlet(1)] permuted) -- per-kernel device times."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import paper_1505_04650_b200 as C
g = np.random.default_rng(0)
s, n, r = 60, int(os.environ.get("XN", "200000")), 50
w0 = np.abs(g.standard_normal((s, r)))
h = np.zeros((r, n)); h[:, :r] = np.eye(r); h[:, r:] = g.dirichlet(np.ones(r), size=n - r).T
h = h[:, g.permutation(n)]
red = w0 @ h + 0.01 * g.standard_normal((s, n))
red_d = torch.from_numpy(red).cuda()
C.select_columns_xray(red_d, 5)
torch.cuda.synchronize()
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    picks = C.select_columns_xray(red_d, r)
    torch.cuda.synchronize()
print("wall", time.perf_counter() - t0, "picks", len(picks))
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.replace("(anonymous namespace)", "")[:60]
        agg[k][0] += 1
        agg[k][1] += e.time_range.end - e.time_range.start
print("picks", [int(x) for x in list(picks)[:12]])
nn = [e.time_range.end - e.time_range.start for e in prof.events()
      if e.device_type == torch.autograd.DeviceType.CUDA and "nnls_kernel" in e.name]
print("nnls us per refit:", " ".join(f"{t:.0f}" for t in nn))
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:6]:
    print(f"{t/1e3:10.2f} ms {c:5d} launches {t / c:9.1f} us avg  {k}")
