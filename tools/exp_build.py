"""Time the K1 build (cb_tensor_coeffs) per BASELINE shape with CUDA events: the GPU is kept
busy (sleep kernel) while the host enqueues the build, so the events bracket the kernels only.
Reports warm (L2-resident input) and cold (256 MiB L2 flush before) times, launches per build and
the algorithmic HBM rate 16 n^J bytes / time; also the per-launch kernel times (torch profiler)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2307_04688_b200 import _lib, workloads  # noqa: E402
from paper_2307_04688_b200.chebnd import tensor_coeffs_device  # noqa: E402

res = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lib = _lib.load()
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3", "4", "5a"]
for cfg in cfgs:
    w = workloads.make(cfg, M=16)
    shape = (w.n,) * w.J
    vals = _lib.to_device(w.values)
    L = _lib.eval_layout(shape)
    coef = _lib.empty((L["elems"],))
    for _ in range(3):
        tensor_coeffs_device(vals, shape, out=coef)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    warm, cold = [], []
    launches = 0
    for flushed in (False, True):
        for _ in range(7):
            if flushed:
                flush.zero_()
            torch.cuda._sleep(200_000)
            n0 = lib.cb_kernel_launches()
            e0.record()
            tensor_coeffs_device(vals, shape, out=coef)
            e1.record()
            e1.synchronize()
            (cold if flushed else warm).append(e0.elapsed_time(e1) * 1000)
            launches = lib.cb_kernel_launches() - n0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            tensor_coeffs_device(vals, shape, out=coef)
        torch.cuda.synchronize()
    kern = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = kern.setdefault(ev.name[:70], [0, 0.0])
            k[0] += 1
            k[1] += ev.device_time_total
    b = 16 * w.values.size
    res[cfg] = {"shape": list(shape), "us_warm": min(warm), "us_cold": min(cold), "launches": launches,
                "GBps_warm": b / (min(warm) * 1e-6) / 1e9, "GBps_cold": b / (min(cold) * 1e-6) / 1e9,
                "kernels_us_per_build": {k: round(v[1] / 5, 2) for k, v in kern.items()}}
print(json.dumps(res, indent=1))
