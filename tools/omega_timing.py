"""Device time of the seeded test matrix (Philox + ziggurat, host tail fix-up
node) for configs[1] shapes, eager and as a replayed CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1505_04650_b200 import _lib
from paper_1505_04650_b200.device import empty, stream

lib = _lib.load()
for rows in (5000, 10000):
    out = empty((rows, 32))
    f = lambda: _lib.call("cnmf_gaussian_fill", 12345, rows, 30, 4096, 0, out.data_ptr(), 32, stream())
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"rows {rows}: eager {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"rows {rows}: graph {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
