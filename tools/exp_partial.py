"""K2: cost of the partial last row block -- 17^4 (R8 = 296 = 3 x 96 + 8) against shapes whose rows
divide the 96-row stages exactly, normalised by the DMMA work R8 x Kp per point."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2307_04688_b200 import _lib
from paper_2307_04688_b200.chebnd import tensor_coeffs_device

lib = _lib.load()
M = 1 << 19
res = {}
for shape in ((17, 17, 17, 17), (16, 18, 17, 17), (12, 24, 17, 17), (19, 15, 17, 17)):
    rng = np.random.default_rng(1)
    vals = rng.standard_normal(shape)
    pts = 2.0 * rng.random((M, 4)) - 1.0
    coef = tensor_coeffs_device(_lib.to_device(vals), shape)
    dp = _lib.to_device(pts)
    out = _lib.empty((M,))
    L = _lib.eval_layout(shape)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for rep in range(4):
        if rep == 1:
            ev[0].record()
        lib.cb_eval_points(4, _lib.i64_array(shape), _lib.ptr(coef), M, _lib.ptr(dp), _lib.ptr(out), None, 0, _lib.stream_handle())
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 3
    work = 2.0 * L["R"] * L["K"] * M
    res[str(shape)] = {"R": L["R"], "R8": L["R8"], "ms": round(ms, 3), "dmma_tflops": round(work / ms / 1e9, 2),
                       "plan": lib.cb_last_eval_plan().decode()[:70]}
print(json.dumps(res, indent=1))
