"""Where the configs[4] end-to-end call spends its wall time (host matrix in pinned memory)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1505_04650_b200 as C
from paper_1505_04650_b200.device import DeviceMatrix
cid = 4
c = bench.CONFIGS[cid]
a, _ = bench.device_data(cid, 0, c["n"], 0)
host = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
rows = 1 << 13
for i in range(0, a.shape[0], rows):
    host[i:i + rows].copy_(a[i:i + rows])
torch.cuda.synchronize()
del a
torch.cuda.empty_cache()
cfg = C.CompressionConfig(r=c["r"], r_ov=10, w=c["q"], seed=7)
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, (time.perf_counter() - t0) * 1e3
for rep in range(3):
    A, ms_copy = t(lambda: DeviceMatrix(host))
    fp, ms_job = t(lambda: C.nmf_admm(A.t, c["r"], cfg=cfg, max_iter=c["iters"], tol=1e-4))
    _, ms_d2h = t(lambda: (fp.X.cpu(), fp.Y.cpu()))
    del A
    _, ms_all = t(lambda: C.nmf_admm(host, c["r"], cfg=cfg, max_iter=c["iters"], tol=1e-4))
    print(f"rep {rep}: H2D (alloc + copy) {ms_copy:.0f} ms = {host.numel() * 4 / ms_copy / 1e6:.1f} GB/s | job on the device copy {ms_job:.0f} ms | D2H of the factors {ms_d2h:.0f} ms | whole call on the host matrix {ms_all:.0f} ms", flush=True)
