"""ncu driver for the structured evaluation (config 5a): one build + eval_grid after warm-up."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2307_04688_b200 as cn
from paper_2307_04688_b200 import _lib, workloads

w = workloads.make("5a")
bases = [cn.make_basis(w.n - 1, 0.0, 1.0)] * w.J
vals = _lib.to_device(w.values)
tdev = [_lib.to_device(t) for t in w.targets]
for _ in range(3):
    out = cn.eval_grid(cn.tensor_coeffs(vals, bases), tdev)
torch.cuda.synchronize()
print("ok", float(out[0, 0, 0, 0, 0, 0]))
