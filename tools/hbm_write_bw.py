"""DRAM bandwidth of a pure write stream (fill) vs a copy on this GPU: the ceiling for write-bound
kernels such as the last K3 pass."""
import torch
x = torch.empty(2 * 1024**3 // 8, dtype=torch.float64, device="cuda")  # 2 GB
y = torch.empty_like(x)
for name, fn in (("fill (write only)", lambda: x.fill_(1.0)), ("copy (read+write)", lambda: y.copy_(x))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(5):
        e0.record(); fn(); e1.record(); e1.synchronize(); ms.append(e0.elapsed_time(e1))
    b = x.numel() * 8 * (1 if "fill" in name else 2)
    print(name, "%.1f GB/s" % (b / (min(ms) * 1e-3) / 1e9))
