import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
from dataclasses import replace
import numpy as np, torch
import cnmf_oracle as O
import paper_1505_04650_b200 as C
from paper_1505_04650_b200 import distributed as D
from paper_1505_04650_b200.device import DeviceMatrix
a32 = O.dense_lowrank(2000, 1001, 20, 0.01, seed=0).astype(np.float32)
a = a32.astype(np.float64)
m, n = a.shape
ops, comm = D.DeviceOps(), D.Comm()
A = DeviceMatrix(torch.from_numpy(a32).cuda())
# orthonormalisation pieces
P = torch.randn(1001, 32, device="cuda"); P[:, 30:] = 0
D.orthonormalize_sharded(ops, comm, P, 30, 32)
q = P[:, :30].double()
print("sharded CholQR2 orth err", (q.t() @ q - torch.eye(30, device="cuda", dtype=torch.float64)).abs().max().item(),
      "pad", P[:, 30:].abs().max().item())
P = torch.randn(2000, 32, device="cuda"); P[:, 30:] = 0
ops.orthonormalize(P, 30)
q = P[:, :30].double()
print("orthonormalize err", (q.t() @ q - torch.eye(30, device="cuda", dtype=torch.float64)).abs().max().item())
cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), m, n)
lc = replace(cfg, seed=O.child_seed(5, "left-basis"))
oc = O.adjust(O.Config(20, 10, 4, O.child_seed(5, "left-basis")), m, n)
Lref = O.range_basis(a, oc)
Ld = D.range_finder(ops, comm, A, m, n, 0, lc, 0)[:, :30].double().cpu().numpy()
Ls = C.structured_compress(a32, lc).Q
print("dist vs oracle", O.projector_distance(Lref, Ld), "single vs oracle", O.projector_distance(Lref, Ls),
      "dist vs single", O.projector_distance(Ld, Ls))
for w in (0, 1, 2):
    oc2 = replace(oc, w=w); lc2 = replace(lc, w=w)
    Lref = O.range_basis(a, oc2)
    Ld = D.range_finder(ops, comm, A, m, n, 0, lc2, 0)[:, :30].double().cpu().numpy()
    print("w", w, "dist vs oracle", O.projector_distance(Lref, Ld), "single", O.projector_distance(Lref, C.structured_compress(a32, lc2).Q))
