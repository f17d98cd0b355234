"""Minimal driver for ncu: one build + one evaluation of a BASELINE config after warm-up.

  python tools/prof_eval.py --config 2 [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2307_04688_b200 import _lib, workloads  # noqa: E402
from paper_2307_04688_b200.chebnd import _eval_points_device, tensor_coeffs_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--M", type=int, default=None)
args = ap.parse_args()

w = workloads.make(args.config, M=args.M)
shape = (w.n,) * w.J
vals = _lib.to_device(w.values)
L = _lib.eval_layout(shape)
coef = _lib.empty((L["elems"],))
if w.points is not None:
    pts = _lib.to_device(w.points)
    out = _lib.empty((w.points.shape[0],))
    for _ in range(args.reps):
        tensor_coeffs_device(vals, shape, out=coef)
        _eval_points_device(shape, coef, pts, check=False, out=out)
else:
    lib = _lib.load()
    N = w.n ** w.J
    out = _lib.empty((N,))
    for _ in range(args.reps):
        tensor_coeffs_device(vals, shape, out=coef)
        lib.cb_eval_advected(w.J, _lib.i64_array(shape), _lib.ptr(coef), 0, N, _lib.dbl_array(w.A), w.dt,
                             _lib.dbl_array([0.0] * w.J), _lib.dbl_array([1.0] * w.J), 1, _lib.ptr(out),
                             _lib.stream_handle())
torch.cuda.synchronize()
print("ok", float(_lib.to_host(out)[:4].sum()))
