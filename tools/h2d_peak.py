"""Host->device copy bandwidth from pinned memory (the e2e path's ceiling)."""
import torch

n = 1 << 30  # 4 GiB of fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for chunk in (1 << 24, 1 << 26, 1 << 28, n):
    s = torch.cuda.Stream()
    d[:chunk].copy_(h[:chunk], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for off in range(0, n, chunk):
        d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"chunk {chunk * 4 >> 20} MiB: {n * 4 / ms / 1e6:.1f} GB/s")
