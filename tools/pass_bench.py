"""Time the streaming passes alone on a configs[1]-shaped A (m x n fp32):
whole call (split panel + memset + kernel) and the pass kernel alone."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros

M, N, S = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10000, 5000, 32)))
reps = int(os.environ.get("REPS", "20"))
lib = _lib.load()
a = torch.rand(M, N, device="cuda")
A = DeviceMatrix(a)
X = torch.randn(N, S, device="cuda")
W = torch.randn(M, S, device="cuda")
Y = zeros((M, S))
Z = zeros((N, S))
for impl in [int(x) for x in os.environ.get("IMPL", "1,0").split(",")]:
    lib.cnmf_set_pass_impl(impl)
    for name, fn in (("forward", lambda: lib.cnmf_pass_forward(A.ptr, M, N, A.lda, X.data_ptr(), S, Y.data_ptr(), stream())),
                     ("transpose", lambda: lib.cnmf_pass_transpose(A.ptr, M, N, A.lda, W.data_ptr(), S, Z.data_ptr(), stream()))):
        for _ in range(3):
            st_ = fn()
            if st_ != 0:
                raise SystemExit(f"status {st_}: {lib.cnmf_last_error()}")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        lib.cnmf_set_pass_profiling(1)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        kms, kl, kby = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        lib.cnmf_pass_stats(ctypes.byref(kms), ctypes.byref(kl), ctypes.byref(kby))
        lib.cnmf_set_pass_profiling(0)
        k = kms.value / max(kl.value, 1)
        print(f"impl={'tc' if impl else 'ffma'} {name:9s} call {ms*1e3:7.1f} us {4*M*N/ms/1e6:7.1f} GB/s | "
              f"kernel {k*1e3:7.1f} us {4*M*N/k/1e6:7.1f} GB/s", flush=True)
