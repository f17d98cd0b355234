"""Device time of one Bellman sweep kernel and one refit, separately (CUDA events, 200 reps)."""
import ctypes, os, sys, warnings
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2307_04688_b200 as cn
from paper_2307_04688_b200 import _lib
from paper_2307_04688_b200.solver import _Device

for preset, kw in (("example1", dict(tol=1e-8)), ("example3", {}), ("example4", {})):
    spec = cn.preset_spec(preset, **kw)
    grid = cn.build_state_grid(spec)
    stacks = cn.precompute_dynamics_stack(spec, grid)
    dev = _Device(spec, grid, stacks)
    J, n = spec.J, grid.n_nodes
    v = _lib.to_device(np.zeros((J, n)))
    u = _lib.to_device(np.broadcast_to(spec.A[:, None], (J, n)).copy())
    coef = _lib.empty((J, n)); dev.refit(v, coef)
    vo, uo = _lib.empty((J, n)), _lib.empty((J, n))
    cl = torch.zeros(1, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    def sweep():
        lib.cb_bellman_sweep(ctypes.byref(dev.game), _lib.ptr(dev.nodes), _lib.ptr(dev.drift), _lib.ptr(coef),
                             _lib.ptr(v), _lib.ptr(u), _lib.ptr(vo), _lib.ptr(uo), _lib.ptr(cl), None,
                             _lib.stream_handle())
    res = {}
    for name, fn in (("sweep", sweep), ("refit", lambda: dev.refit(vo, coef))):
        for _ in range(10):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 200 * 1000, 1)
    print(preset, "us per launch (back to back, host-launched):", res)
