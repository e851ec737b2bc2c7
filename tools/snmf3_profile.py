"""Per-kernel device times of the whole configs[3] SNMF job (bench.py's generator)."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import bench
import paper_1505_04650_b200 as C
cid = int(os.environ.get("CID", "3"))
c = bench.CONFIGS[cid]
a, truth = bench.device_data(cid, 0, c["n"], 0)
cfg = C.CompressionConfig(r=c["r"], r_ov=10, w=c["q"], seed=7)
res = C.snmf(a, c["r"], selector=c["sel"], cfg=cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = C.snmf(a, c["r"], selector=c["sel"], cfg=cfg)
    torch.cuda.synchronize()
print("wall", time.perf_counter() - t0, "picks ok", sorted(res.K.tolist()) == truth, "rel", res.rel_error_full)
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.replace("(anonymous namespace)", "")[:70]
        agg[k][0] += 1
        agg[k][1] += e.time_range.end - e.time_range.start
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{t/1e3:10.2f} ms {n:5d} launches {t / n:9.1f} us avg  {k}")
nn = [e.time_range.end - e.time_range.start for e in prof.events()
      if e.device_type == torch.autograd.DeviceType.CUDA and "nnls_kernel" in e.name]
print("nnls us per launch:", " ".join(f"{t:.0f}" for t in nn))
