"""Time cb_eval_grid (config 5a shape) on symmetric (linspace) and non-symmetric targets."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_04688_b200 as cn  # noqa: E402
from paper_2307_04688_b200 import _lib, workloads  # noqa: E402
from paper_2307_04688_b200.chebnd import _eval_grid_device, tensor_coeffs_device  # noqa: E402

w = workloads.make("5a")
shape = (13,) * 6
coef = tensor_coeffs_device(_lib.to_device(w.values), shape)
rng = np.random.default_rng(1)
sym = [(2.0 * np.arange(25) - 24.0) / 24.0 for _ in range(6)]   # exactly symmetric uniform grid
for name, targets in (("linspace", w.targets), ("symmetric", sym),
                      ("nonsymmetric", [np.sort(2 * rng.random(25) - 1) for _ in range(6)])):
    tdev = [_lib.to_device(t) for t in targets]
    sym_flag = all(np.array_equal(np.asarray(t)[::-1], -np.asarray(t)) for t in targets)
    st = _lib.new_status()
    out = _lib.empty((25,) * 6)
    for _ in range(3):
        _eval_grid_device(shape, coef, tdev, status=st, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(5):
        torch.cuda._sleep(400_000)
        e0.record()
        _eval_grid_device(shape, coef, tdev, status=st, out=out)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(name, "symmetric" if sym_flag else "plain", "eval_grid ms min %.3f" % min(ms), flush=True)
