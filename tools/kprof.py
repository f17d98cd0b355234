"""Per-kernel device times (torch.profiler / CUPTI) for one workload's hot call, after warm-up.
Usage: python tools/kprof.py {5a|5b|2|3|4|build4|build2}"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2307_04688_b200 as cn
from paper_2307_04688_b200 import _lib, workloads

which = sys.argv[1] if len(sys.argv) > 1 else "5a"
key = which.replace("build", "")
w = workloads.make(key, M=None) if key in ("2", "4") else workloads.make(key)
bases = [cn.make_basis(n - 1, 0.0, 1.0) for n in w.values.shape]
vals = _lib.to_device(w.values)
if which.startswith("build"):
    from paper_2307_04688_b200.chebnd import tensor_coeffs_device
    shp = tuple(w.values.shape)
    fn = lambda: tensor_coeffs_device(vals, shp)
elif which == "5a":
    t = cn.tensor_coeffs(vals, bases)
    tdev = [_lib.to_device(x) for x in w.targets]
    fn = lambda: cn.eval_grid(t, tdev)
else:
    t = cn.tensor_coeffs(vals, bases)
    pts = _lib.to_device(w.points)
    fn = lambda: cn.eval_points(t, pts)
for _ in range(3):
    fn()
torch.cuda.synchronize()
reps = 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
rows = {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        r = rows.setdefault(ev.name[:90], [0, 0.0])
        r[0] += 1
        r[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = 0.0
for name, (cnt, us) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
    print(f"{us / reps:10.1f} us/call  x{cnt // reps:<3d} {name}")
    tot += us / reps
print(f"{tot:10.1f} us total per call")
