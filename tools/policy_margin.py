"""Max |policy - reference| of the GPU solver on the golden solver fixtures (sweep and full solve)."""
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2307_04688_b200 as cn  # noqa: E402
from test_gpu_solver import GOLD, KEYS, spec_of  # noqa: E402

for key in KEYS:
    spec = spec_of(key)
    grid = cn.build_state_grid(spec)
    stacks = cn.precompute_dynamics_stack(spec, grid)
    v0, u0 = GOLD[f"{key}_sweep_v0"], GOLD[f"{key}_sweep_u0"]
    interp = [cn.tensor_coeffs(v0[i].reshape(grid.shape, order="F"), grid.bases) for i in range(spec.J)]
    vf, pf = cn.bellman_sweep(spec, grid, cn.ValueField(v0, interp), cn.PolicyField(u0), stacks)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        res = cn.solve(spec)
    print(key, "sweep policy max|d| %.3e" % np.abs(pf.values - GOLD[f"{key}_sweep_u1"]).max(),
          "solve policy max|d| %.3e" % np.abs(res.policy.values - GOLD[f"{key}_solve_policy"]).max(),
          "solve values max|d| %.3e" % np.abs(res.values.values - GOLD[f"{key}_solve_values"]).max(),
          "U_max", spec.U_max, flush=True)
