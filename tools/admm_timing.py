"""Per-iteration cost of the persistent ADMM kernel on configs[1] shapes."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_04650_b200 as C
from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros
from paper_1505_04650_b200.nmf import compressed_problem
from paper_1505_04650_b200.rng import Rng
M, N, R = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10000, 5000, 20)))
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.addmm(0.01 * torch.randn(M, N, device="cuda", generator=g), torch.rand(M, R, device="cuda", generator=g),
                torch.rand(R, N, device="cuda", generator=g)).clamp_(min=0)
A = DeviceMatrix(a)
cfg = C.adjust_config(C.CompressionConfig(r=R, r_ov=10, w=4, seed=5), M, N)
s = cfg.basis_cols
left, right, core = compressed_problem(A, cfg)
lib = _lib.load()
rng = Rng(cfg.seed)
u0 = rng.child("init-left").uniform((M, R)); vt0 = rng.child("init-right").uniform((R, N), transpose=True)
du = zeros((M, R), torch.float64); dvt = zeros((N, R), torch.float64)
xc = zeros((s, R), torch.float64); yc = zeros((R, s), torch.float64)
trace = zeros((1000,), torch.float64); scores = zeros((1000,), torch.float64)
nb = lib.cnmf_admm_workspace(M, N, s, R); ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
it = ctypes.c_int(0); done = ctypes.c_int(0)
for iters in [int(x) for x in os.environ.get("ITERS", "1,10,100,500").split(",")]:
    ts = []
    for rep in range(3):
        u = u0.clone(); vt = vt0.clone()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = lib.cnmf_admm_run(core.data_ptr(), left.panel.data_ptr(), M, right.panel.data_ptr(), N, s, R, u.data_ptr(),
                               du.data_ptr(), vt.data_ptr(), dvt.data_ptr(), xc.data_ptr(), yc.data_ptr(), 1.0, 1.0, 1.0,
                               iters, 0.0, trace.data_ptr(), scores.data_ptr(), ctypes.byref(it), ctypes.byref(done), 0, 0,
                               ws.data_ptr(), nb, stream())
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        _lib.check(st)
    print(f"iters={iters:4d} best {min(ts)*1e3:8.3f} ms  per-iter {min(ts)/iters*1e6:8.2f} us  done={it.value}")
