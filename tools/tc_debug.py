import sys, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros
lib = _lib.load()
for (m, n) in [(128, 32), (256, 64), (1000, 700)]:
    for mode in ("ones", "rand"):
        g = np.random.default_rng(0)
        a = np.ones((m, n)) if mode == "ones" else g.standard_normal((m, n))
        x = np.zeros((n, 32), np.float32); x[:, :30] = 1.0 if mode == "ones" else g.standard_normal((n, 30))
        A = DeviceMatrix(a); X = torch.from_numpy(x).cuda(); Y = zeros((m, 32))
        st = lib.cnmf_pass_forward(A.ptr, m, n, A.lda, X.data_ptr(), 30, Y.data_ptr(), stream())
        torch.cuda.synchronize()
        y = Y.cpu().numpy(); ref = a.astype(np.float32).astype(np.float64) @ x
        print(m, n, mode, 'status', st, 'y[0,:4]', y[0, :4], 'ref', ref[0, :4], 'max|y|', np.abs(y).max(),
              'relerr', np.linalg.norm(y - ref) / np.linalg.norm(ref))
        W = torch.from_numpy(x[:1, :].repeat(m, 0) if False else np.zeros((m, 32), np.float32)).cuda()
print(torch.cuda.synchronize())
