"""H2D bandwidth of a pinned host buffer: one copy vs chunked copies on 1-4 streams."""
import time
import torch
n = 16 * (1 << 30) // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for streams, chunks in ((1, 1), (1, 8), (2, 8), (4, 16), (2, 32)):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = n // chunks
    for i in range(chunks):
        with torch.cuda.stream(ss[i % streams]):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"streams {streams} chunks {chunks}: {4 * n / dt / 1e9:.1f} GB/s", flush=True)
