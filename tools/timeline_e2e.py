"""Device timeline of one e2e call of the public API with pinned host buffers (config 2 by
default): H2D copies, build, chunked evaluation, D2H copies and the gaps between them."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2307_04688_b200 as cn
from paper_2307_04688_b200 import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
w = workloads.make(cfg)
bases = [cn.make_basis(w.n - 1, 0.0, 1.0)] * w.J
vals = torch.from_numpy(np.ascontiguousarray(w.values)).pin_memory()
pts = torch.from_numpy(np.ascontiguousarray(w.points)).pin_memory()
for _ in range(3):
    cn.eval_points(cn.tensor_coeffs(vals, bases), pts)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    cn.eval_points(cn.tensor_coeffs(vals, bases), pts)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
for e in ev:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    print(f"{s - t0:9.1f} us  gap {s - prev_end:7.1f}  dur {d:8.1f}  {e.name[:90]}")
    prev_end = max(prev_end, s + d)
print(f"device span {prev_end - t0:.1f} us")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
if cpu:
    print(f"host span {max(e.time_range.end for e in cpu) - min(e.time_range.start for e in cpu):.1f} us")
