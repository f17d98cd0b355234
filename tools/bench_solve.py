"""Time-to-solution of the device solver on the reference's acceptance workloads
(T/test_acceptance.py #6-#8 and the example1 tol=1e-8 fixture), plus the CPU oracle's per-sweep
time on the same specs (bounded sample of sweeps, extrapolated).  Prints one JSON line per case."""
import json
import os
import sys
import time
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2307_04688_b200 as cn  # noqa: E402

CASES = [
    ("example1_tol1e-8", "example1", dict(tol=1e-8)),
    ("example1_deg4", "example1", dict(Np=4, Nu=4)),
    ("example3", "example3", {}),
    ("example4", "example4", {}),
    ("example3_np7_h1e-2", "example3", dict(Np=7, Nu=7, h=1e-2, tol=1e-3, max_iters=20_000)),
]

cpu = "--cpu" in sys.argv
only = [a for a in sys.argv[1:] if not a.startswith("--")]
for name, preset, kw in CASES:
    if only and name not in only:
        continue
    spec = cn.preset_spec(preset, **kw)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        cn.solve(cn.preset_spec(preset, **{**kw, "max_iters": 3}))  # warm-up (graph + modules)
        t0 = time.perf_counter()
        res = cn.solve(spec)
        wall = time.perf_counter() - t0
    line = {"case": name, "J": spec.J, "nodes": int(np.prod(spec.Np + 1)), "converged": res.converged,
            "iterations": res.iterations, "wall_s": wall, "sweeps_per_s": res.iterations / res.timings["sweeps"],
            "us_per_sweep": 1e6 * res.timings["sweeps"] / res.iterations}
    if cpu:
        from oracle import solver_oracle as so

        g = so.Game(J=spec.J, K=np.asarray(spec.K), beta=spec.beta, phi=spec.phi, A=spec.A, c=spec.c, m=spec.m,
                    rho=spec.rho, h=spec.h, P_max=spec.P_max, U_max=spec.U_max, Np=spec.Np, Nu=spec.Nu, tol=spec.tol,
                    max_iters=spec.max_iters)
        S = so.Solver(g)
        n_s = 20
        t0 = time.perf_counter()
        S.solve(max_iters=n_s)
        per = (time.perf_counter() - t0) / n_s
        line.update(cpu_s_per_sweep=per, cpu_extrapolated_s=per * res.iterations,
                    speedup=per * res.iterations / wall)
    print(json.dumps(line), flush=True)
