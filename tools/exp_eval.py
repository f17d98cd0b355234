"""Timing experiments on the K2 evaluator (debug switches of cb_eval_points flags)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2307_04688_b200 import _lib, workloads
from paper_2307_04688_b200.chebnd import tensor_coeffs_device

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
flag_list = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
w = workloads.make(cfg, M=(1 << 20) if cfg in ("2",) else (1 << 19))
shape = (w.n,) * w.J
if w.points is None:  # loop configs (3, 5b): seeded uniform points of the same shape
    import numpy as np
    w.points = 2.0 * np.random.default_rng(7).random(((1 << 19), w.J)) - 1.0
coef = tensor_coeffs_device(_lib.to_device(w.values), shape)
pts = _lib.to_device(w.points)
out = _lib.empty((w.points.shape[0],))
lib = _lib.load()
flops = 2 * sum(w.n ** m for m in range(1, w.J + 1)) * w.points.shape[0]
res = {}
ref = None
for flags in flag_list:
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for rep in range(4):
        if rep == 1:
            ev[0].record()
        lib.cb_eval_points(w.J, _lib.i64_array(shape), _lib.ptr(coef), w.points.shape[0], _lib.ptr(pts), _lib.ptr(out), None, flags, _lib.stream_handle())
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 3
    o = _lib.to_host(out)
    if ref is None:
        ref = o.copy()
    res[flags] = [round(flops / ms / 1e9, 2), bool((o == ref).all()), float(abs(o - ref).max()),
                  lib.cb_last_eval_plan().decode()[:60]]
print(json.dumps({"cfg": cfg, "tflops,bitwise_vs_first,maxabs,plan": res}))
