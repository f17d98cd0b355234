"""Time the K1 build (cb_tensor_coeffs) per BASELINE shape with CUDA events (L2 warm / flushed)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2307_04688_b200 import _lib, workloads
from paper_2307_04688_b200.chebnd import tensor_coeffs_device

res = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lib = _lib.load()
for cfg in ("1", "2", "3", "4", "5a"):
    w = workloads.make(cfg, M=16)
    shape = (w.n,) * w.J
    vals = _lib.to_device(w.values)
    L = _lib.eval_layout(shape)
    coef = _lib.empty((L["elems"],))
    for _ in range(3):
        tensor_coeffs_device(vals, shape, out=coef)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    warm, cold = [], []
    for flushed in (False, True):
        for _ in range(5):
            if flushed:
                flush.zero_()
            n0 = lib.cb_kernel_launches()
            e0.record()
            tensor_coeffs_device(vals, shape, out=coef)
            e1.record()
            e1.synchronize()
            (cold if flushed else warm).append(e0.elapsed_time(e1) * 1000)
            launches = lib.cb_kernel_launches() - n0
    b = 16 * w.values.size
    res[cfg] = {"us_warm": min(warm), "us_cold": min(cold), "launches": launches,
                "GBps_cold": b / (min(cold) * 1e-6) / 1e9}
print(json.dumps(res))
