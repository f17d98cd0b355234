"""Minimal driver for ncu: warm-up then one K1 build of a BASELINE config.
  python tools/prof_build.py --config 5a"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2307_04688_b200 import _lib, workloads  # noqa: E402
from paper_2307_04688_b200.chebnd import tensor_coeffs_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="5a")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
w = workloads.make(args.config, M=16)
shape = (w.n,) * w.J
vals = _lib.to_device(w.values)
coef = _lib.empty((_lib.eval_layout(shape)["elems"],))
for _ in range(args.reps):
    tensor_coeffs_device(vals, shape, out=coef)
torch.cuda.synchronize()
print("ok")
