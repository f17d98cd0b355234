"""Device timeline of one device-resident step (kernels, copies, gaps) via torch.profiler (CUPTI).

    python tools/timeline.py 5a      # build + eval_grid (config 5a)
    python tools/timeline.py 2       # build + eval_points (config 2)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2307_04688_b200 as cn  # noqa: F401
from paper_2307_04688_b200 import _lib, workloads
from paper_2307_04688_b200.chebnd import _eval_grid_device, _eval_points_device, tensor_coeffs_device

cfg = sys.argv[1] if len(sys.argv) > 1 else "5a"
w = workloads.make(cfg)
shape = (w.n,) * w.J
vals = _lib.to_device(w.values)
L = _lib.eval_layout(shape)
coef = _lib.empty((L["elems"],))
st = _lib.new_status()
if cfg == "5a":
    tdev = [_lib.to_device(t) for t in w.targets]
    out = _lib.empty(tuple(int(t.shape[0]) for t in tdev))

    def step():
        tensor_coeffs_device(vals, shape, out=coef, status=st)
        _eval_grid_device(shape, coef, tdev, status=st, out=out)
else:
    pts = _lib.to_device(w.points)
    out = _lib.empty((pts.shape[0],))

    def step():
        tensor_coeffs_device(vals, shape, out=coef, status=st)
        _eval_points_device(shape, coef, pts, check=False, out=out)

for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
for e in ev:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    print(f"{s - t0:9.1f} us  gap {s - prev_end:7.1f}  dur {d:8.1f}  {e.name[:100]}")
    prev_end = max(prev_end, s + d)
print(f"total {prev_end - t0:.1f} us")
