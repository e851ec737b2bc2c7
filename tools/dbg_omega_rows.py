import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import numpy as np, torch
import cnmf_oracle as O
from paper_1505_04650_b200 import distributed as D
from paper_1505_04650_b200.rng import child_seed
ops = D.DeviceOps()
seed = O.child_seed(O.child_seed(5, "left-basis"), "omega")
full = O.test_matrix(5000, 30, O.child_seed(5, "left-basis"))
for row0, rows in ((0, 1001), (4000, 200), (4096, 100)):
    got = ops.omega_rows(seed, row0, rows, 30, 32)[:, :30].double().cpu().numpy()
    ref = full[row0:row0+rows]
    print(row0, rows, np.abs(got - ref).max(), got[0,:3], ref[0,:3])
print(child_seed(5, "left-basis"), O.child_seed(5, "left-basis"))
