"""Generate tests/golden/golden_solver_v1.npz by running the REFERENCE solver itself (SURVEY.md
§8f row 1: the Bellman sweep / `solve`, plus `newton_maximize`, the drift stacks and `simulate`).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_solver.py

Every array stored here is an output of the reference's public (or solver-private) functions on
seeded inputs.  The fixtures pin the CPU solver restatement (oracle/solver_oracle.py) and the CUDA
sweep (tests/test_gpu_solver.py); /root/reference does not travel to the GPU box.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("CHEBNASH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import chebnash as ref  # noqa: E402
from chebnash import solver as rs  # noqa: E402

# the reference test-suite's fast settings (T/test_solver.py:25)
FAST = dict(rho=0.5, h=0.01, P_max=0.5, U_max=0.5, tol=1e-6, max_iters=20_000)

# (key, preset, overrides) of the specs whose sweeps / solves are pinned
SPECS = [
    ("e1a", "example1", dict(FAST, Np=2, Nu=3)),
    ("e1b", "example1", dict(FAST, Np=3, Nu=3)),
    ("e1c", "example1", dict(FAST, Np=4, Nu=5, tol=1e-8)),
    ("e3a", "example3", dict(FAST, Np=2, Nu=2, tol=1e-8)),
    ("e4a", "example4", dict(FAST, Np=2, Nu=3, tol=1e-4)),
    ("e1d", "example1", dict(FAST, Np=2, Nu=2, tol=1e-4)),
]


def spec_arrays(key, spec, out):
    out[f"{key}_spec_K"] = np.asarray(spec.K)
    for name in ("beta", "phi", "A", "c", "m", "Np", "Nu"):
        out[f"{key}_spec_{name}"] = np.asarray(getattr(spec, name))
    out[f"{key}_spec_scalars"] = np.array([spec.J, spec.rho, spec.h, spec.P_max, spec.U_max, spec.tol,
                                           spec.max_iters], dtype=float)


def quiet_solve(spec, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return ref.solve(spec, **kw)


def main():
    out = {}
    rng = np.random.default_rng(20240807)
    for key, preset, kw in SPECS:
        spec = ref.preset_spec(preset, **kw)
        spec_arrays(key, spec, out)
        grid = ref.build_state_grid(spec)
        stacks = ref.precompute_dynamics_stack(spec, grid)
        for i, st in enumerate(stacks):
            out[f"{key}_stack{i}"] = np.asarray(st.coefficients)
        # one sweep from a seeded random state (values + feasible policy)
        n = grid.n_nodes
        shape = grid.shape
        v0 = 0.01 * rng.standard_normal((spec.J, n))
        u0 = rng.uniform(0.0, spec.U_max, (spec.J, n))
        interp = [ref.tensor_coeffs(v0[i].reshape(shape, order="F"), grid.bases) for i in range(spec.J)]
        vf = rs.ValueField(values=v0, interpolants=interp)
        pf = rs.PolicyField(values=u0)
        v1, u1 = rs.bellman_sweep(spec, grid, vf, pf, stacks)
        out[f"{key}_sweep_v0"] = v0
        out[f"{key}_sweep_u0"] = u0
        out[f"{key}_sweep_v1"] = v1.values
        out[f"{key}_sweep_u1"] = u1.values
        out[f"{key}_sweep_c1"] = np.stack([t.coefficients for t in v1.interpolants])
        # full solve from the default initial fields
        res = quiet_solve(spec)
        out[f"{key}_solve_converged"] = np.array(res.converged)
        out[f"{key}_solve_iterations"] = np.array(res.iterations)
        out[f"{key}_solve_values"] = res.values.values
        out[f"{key}_solve_policy"] = res.policy.values
        out[f"{key}_solve_history"] = res.history
        out[f"{key}_solve_clamp"] = np.array(res.clamp_fraction)
        out[f"{key}_solve_coef"] = np.stack([t.coefficients for t in res.values.interpolants])
        print(key, spec.J, n, "iterations", res.iterations, res.converged)
        if key == "e1b":
            pols = ref.fit_policy(grid, res.policy)
            out[f"{key}_fitpolicy"] = np.stack([p.coefficients for p in pols])
            p0 = np.array([0.05, 0.3])
            path = ref.simulate(spec, pols, p0, 500)
            out[f"{key}_sim_p0"] = p0
            out[f"{key}_sim_states"] = path.states
            out[f"{key}_sim_controls"] = path.controls
            out[f"{key}_sim_payoff"] = ref.discounted_payoff(spec, path.states, path.controls, 400)

    # non-convergence and the clamp warning (T/test_solver.py:284-297)
    spec = ref.preset_spec("example1", **dict(FAST, Np=2, Nu=2, P_max=0.2, U_max=0.5, tol=1e-2, max_iters=50))
    spec_arrays("clamp", spec, out)
    res = quiet_solve(spec)
    out["clamp_solve_clamp"] = np.array(res.clamp_fraction)
    out["clamp_solve_iterations"] = np.array(res.iterations)
    out["clamp_solve_values"] = res.values.values
    out["clamp_solve_policy"] = res.policy.values

    # the 1-D maximiser on seeded coefficient rows (T/test_solver.py:139-160) incl. multimodal ones
    basis = ref.make_basis(6, 0.0, 1.0)
    rows = rng.standard_normal((40, 7))
    rows[20:] *= np.array([0.1, 0.2, 1.0, 0.1, 2.0, 0.1, 1.5])  # wigglier rows -> scan fallback
    u0s = rng.uniform(0.0, 1.0, 40)
    res_u, res_f = [], []
    for r, u0 in zip(rows, u0s):
        u, f = ref.newton_maximize(ref.CoefVector(r, basis), float(u0))
        res_u.append(u)
        res_f.append(f)
    out["newton_rows"] = rows
    out["newton_u0"] = u0s
    out["newton_u"] = np.array(res_u)
    out["newton_f"] = np.array(res_f)
    # the block maximiser without the forced scan (the sweep's form), several degrees
    for L in (2, 3, 5, 9):
        c = rng.standard_normal((64, L))
        x0 = rng.uniform(-1.0, 1.0, 64)
        xb, fb = rs._maximise_block(c, x0)
        out[f"maxblock{L}_coef"] = c
        out[f"maxblock{L}_x0"] = x0
        out[f"maxblock{L}_x"] = xb
        out[f"maxblock{L}_f"] = fb

    # the closed-form LQ oracle (S/oracle.py): full solves and one exact update from a random state
    from chebnash import oracle as ro

    for key, preset, kw in (("lq1", "example1", dict(FAST, Np=2, Nu=2)), ("lq2", "example1", {}),
                            ("lq3", "example3", dict(FAST)), ("lq4", "example4", {})):
        spec = ref.preset_spec(preset, **kw)
        spec_arrays(key, spec, out)
        fb = ro.lq_solve(spec)
        for name in ("Q", "b", "d", "e", "f"):
            out[f"{key}_{name}"] = np.asarray(getattr(fb, name))
        out[f"{key}_iterations"] = np.array(fb.iterations)
        out[f"{key}_negfrac"] = np.array(fb.negative_fraction)
        out[f"{key}_highfrac"] = np.array(fb.high_fraction)
        J = spec.J
        st = [0.01 * rng.standard_normal((J, J, J)), 0.01 * rng.standard_normal((J, J)),
              0.01 * rng.standard_normal(J), rng.uniform(0.1, 0.4, J), 0.1 * rng.standard_normal((J, J))]
        st[0] = 0.5 * (st[0] + np.transpose(st[0], (0, 2, 1)))
        upd = ro.lq_bellman_update(spec, *st)
        for name, a, b in zip(("Q", "b", "d", "e", "f"), st, upd):
            out[f"{key}_upd_in_{name}"] = a
            out[f"{key}_upd_out_{name}"] = b
        print(key, "lq iterations", fb.iterations, fb.negative_fraction)
    # policy error of the e1b solve against its oracle (acceptance #6 machinery)
    spec = ref.preset_spec("example1", **dict(FAST, Np=3, Nu=3))
    grid = ref.build_state_grid(spec)
    res = quiet_solve(spec)
    out["perr_e1b"] = np.array(ro.policy_error(res.policy, ro.lq_solve(spec, grid), grid))

    np.savez_compressed(os.path.join(HERE, "golden_solver_v1.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
