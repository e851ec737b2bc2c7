"""Per-launch device times of the CholeskyQR kernels on a tall panel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import stream

rows, s = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (10000, 30)))
lib = _lib.load()
S = lib.cnmf_panel_ld(s)
p = torch.randn(rows, S, device="cuda")
p[:, s:] = 0
R = torch.zeros(S, S, dtype=torch.float64, device="cuda")
nb = 1 << 20
ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
for _ in range(3):
    q = p.clone()
    _lib.call("cnmf_orthonormalize", q.data_ptr(), rows, s, R.data_ptr(), ws.data_ptr(), nb, stream())
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    q = p.clone()
    _lib.call("cnmf_orthonormalize", q.data_ptr(), rows, s, R.data_ptr(), ws.data_ptr(), nb, stream())
    torch.cuda.synchronize()
for e in sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                key=lambda e: e.time_range.start):
    print(f"{e.time_range.end - e.time_range.start:8.1f} us  {e.name[:60]}")
print("orthogonality", (q[:, :s].double().t() @ q[:, :s].double() - torch.eye(s, device='cuda', dtype=torch.float64)).abs().max().item())
