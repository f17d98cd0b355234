"""GPU: the device collocation solver (cb_solver.cu through paper_2307_04688_b200.solver) against
the reference solver's own outputs (tests/golden/golden_solver_v1.npz) and the reference test
suite's solver properties (T/test_solver.py, T/test_acceptance.py #5, #8).

Tolerances: the north star's allclose(rtol=1e-12, atol=1e-11) for values AND policies (policies
are argmax locations of fitted objectives; measured max |difference| on the six golden solves is
6.2e-14, tools/policy_margin.py); the maximiser on identical coefficient rows is bitwise.
"""

import os
import warnings

import numpy as np
import pytest

import paper_2307_04688_b200 as cn
from oracle import solver_oracle as so

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_solver_v1.npz"))
KEYS = ["e1a", "e1b", "e1c", "e3a", "e4a", "e1d"]
FAST = dict(rho=0.5, h=0.01, P_max=0.5, U_max=0.5, tol=1e-6, max_iters=20_000)
RTOL, ATOL = 1e-12, 1e-11


def spec_of(key):
    g = so.game_from_golden(GOLD, key)
    return cn.GameSpec(J=g.J, K=g.K, beta=g.beta, phi=g.phi, A=g.A, c=g.c, m=g.m, rho=g.rho, h=g.h, P_max=g.P_max,
                       U_max=g.U_max, Np=g.Np, Nu=g.Nu, tol=g.tol, max_iters=g.max_iters)


def quiet(fn, *a, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return fn(*a, **kw)


@pytest.mark.parametrize("L", [2, 3, 5, 9])
def test_maximiser_rows_bitwise_vs_reference(cuda, L):
    x, f = cn.solver._maximise_rows(GOLD[f"maxblock{L}_coef"], GOLD[f"maxblock{L}_x0"])
    assert np.array_equal(x, GOLD[f"maxblock{L}_x"]), np.abs(x - GOLD[f"maxblock{L}_x"]).max()
    assert np.array_equal(f, GOLD[f"maxblock{L}_f"]), np.abs(f - GOLD[f"maxblock{L}_f"]).max()


def test_newton_maximize_vs_reference(cuda):
    basis = cn.make_basis(6, 0.0, 1.0)
    for r, u0, ue, fe in zip(GOLD["newton_rows"], GOLD["newton_u0"], GOLD["newton_u"], GOLD["newton_f"]):
        u, f = cn.newton_maximize(cn.CoefVector(r, basis), u0)
        assert u == ue and f == fe


def test_newton_known_answers(cuda):
    # T/test_solver.py:125-136
    b = cn.make_basis(4, 0.0, 1.0)
    c = cn.coeffs_from_samples(b.nodes * (0.5 - b.nodes / 2), b)
    u, val = cn.newton_maximize(c, 0.9)
    assert abs(u - 0.5) < 1e-10 and abs(val - 0.125) < 1e-12
    b3 = cn.make_basis(3, 0.0, 1.0)
    c = cn.coeffs_from_samples(-2.0 * b3.nodes + 0.1 * b3.nodes ** 2, b3)
    u, val = cn.newton_maximize(c, 0.5)
    assert u == 0.0 and abs(val) < 1e-12


@pytest.mark.parametrize("key", KEYS)
def test_drift_stacks_vs_reference(cuda, key):
    spec = spec_of(key)
    stacks = cn.precompute_dynamics_stack(spec, cn.build_state_grid(spec))
    for i, st in enumerate(stacks):
        np.testing.assert_allclose(st.coefficients, GOLD[f"{key}_stack{i}"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("key", KEYS)
def test_bellman_sweep_vs_reference(cuda, key):
    spec = spec_of(key)
    grid = cn.build_state_grid(spec)
    stacks = cn.precompute_dynamics_stack(spec, grid)
    v0, u0 = GOLD[f"{key}_sweep_v0"], GOLD[f"{key}_sweep_u0"]
    interp = [cn.tensor_coeffs(v0[i].reshape(grid.shape, order="F"), grid.bases) for i in range(spec.J)]
    vf, pf = cn.bellman_sweep(spec, grid, cn.ValueField(v0, interp), cn.PolicyField(u0), stacks)
    np.testing.assert_allclose(vf.values, GOLD[f"{key}_sweep_v1"], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(pf.values, GOLD[f"{key}_sweep_u1"], rtol=RTOL, atol=ATOL)
    got_c = np.stack([t.coefficients for t in vf.interpolants])
    np.testing.assert_allclose(got_c, GOLD[f"{key}_sweep_c1"], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("key", KEYS)
def test_solve_vs_reference(cuda, key):
    spec = spec_of(key)
    res = quiet(cn.solve, spec)
    assert res.converged == bool(GOLD[f"{key}_solve_converged"])
    assert res.iterations == int(GOLD[f"{key}_solve_iterations"])
    np.testing.assert_allclose(res.values.values, GOLD[f"{key}_solve_values"], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(res.policy.values, GOLD[f"{key}_solve_policy"], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(res.history, GOLD[f"{key}_solve_history"], rtol=1e-8, atol=1e-13)
    # clamping is decided by the sign of drift values that are zero up to rounding at boundary
    # nodes (|g| ~ 1e-17), so a component or two per sweep may flip; the fraction only feeds the
    # 1 % warning
    assert abs(res.clamp_fraction - float(GOLD[f"{key}_solve_clamp"])) <= 0.02
    got_c = np.stack([t.coefficients for t in res.values.interpolants])
    np.testing.assert_allclose(got_c, GOLD[f"{key}_solve_coef"], rtol=RTOL, atol=ATOL)


def test_clamp_warning_and_non_convergence(cuda):
    spec = cn.preset_spec("example1", **dict(FAST, Np=2, Nu=2, P_max=0.2, U_max=0.5, tol=1e-2, max_iters=50))
    with pytest.warns(RuntimeWarning, match="clamped"):
        res = cn.solve(spec)
    assert res.iterations == int(GOLD["clamp_solve_iterations"])
    assert abs(res.clamp_fraction - float(GOLD["clamp_solve_clamp"])) <= 0.02
    np.testing.assert_allclose(res.values.values, GOLD["clamp_solve_values"], rtol=RTOL, atol=ATOL)
    r5 = quiet(cn.solve, cn.preset_spec("example1", **dict(FAST, Np=2, Nu=2, tol=1e-12, max_iters=5)))
    assert not r5.converged and r5.iterations == 5 and r5.history.shape == (5, 2)


def test_first_sweep_from_zero_recovers_myopic_policy(cuda):
    # T/test_solver.py:167-179
    spec = cn.preset_spec("example1", **dict(FAST, Np=2, Nu=3))
    grid = cn.build_state_grid(spec)
    stacks = cn.precompute_dynamics_stack(spec, grid)
    z = np.zeros((2, grid.n_nodes))
    interp = [cn.tensor_coeffs(np.zeros(grid.shape), grid.bases) for _ in range(2)]
    v1, u1 = cn.bellman_sweep(spec, grid, cn.ValueField(z.copy(), interp), cn.PolicyField(z.copy()), stacks)
    np.testing.assert_allclose(u1.values, 0.5, atol=1e-9)
    for i in range(2):
        expect = spec.delta * spec.h * (0.5 * (0.5 - 0.25) - 0.5 * spec.phi[i] * grid.nodes[:, i] ** 2)
        np.testing.assert_allclose(v1.values[i], expect, atol=1e-12)
    for nb in (3, 9):  # plans never change the result (T/test_solver.py:182-191)
        v, u = cn.bellman_sweep(spec, grid, cn.ValueField(z.copy(), interp), cn.PolicyField(z.copy()), stacks,
                                cn.partition(9, nb))
        assert np.array_equal(v.values, v1.values) and np.array_equal(u.values, u1.values)


def test_solve_properties(cuda):
    # T/test_solver.py:212-281 and acceptance #5
    spec = cn.preset_spec("example1", **dict(FAST, phi=0.0, beta=0.0, rho=1.0, tol=1e-11, max_iters=5000))
    res = quiet(cn.solve, spec)
    assert res.converged
    v_expect = spec.h * spec.delta * 0.5 ** 2 / (2 * (1 - spec.delta))
    np.testing.assert_allclose(res.policy.values, 0.5, atol=1e-8)
    np.testing.assert_allclose(res.values.values, v_expect, atol=1e-8)
    one = quiet(cn.solve, cn.preset_spec("example1", **dict(FAST, tol=10.0)))
    assert one.converged and one.iterations == 1
    sym = quiet(cn.solve, cn.preset_spec("example1", **dict(FAST, Np=4, Nu=4, tol=1e-8)))
    u1 = sym.policy.values[0].reshape(5, 5, order="F")
    u2 = sym.policy.values[1].reshape(5, 5, order="F")
    np.testing.assert_allclose(u1, u2.T, atol=1e-8)
    assert (sym.policy.values >= 0).all() and (sym.policy.values <= 0.5).all()
    tail = sym.history.max(axis=1)[-15:]
    assert np.all(tail[1:] / tail[:-1] <= (1.0 - 0.5 * 0.01) + 0.05)  # contraction (T/test_solver.py:249-256)
    base = quiet(cn.solve, cn.preset_spec("example1", **dict(FAST, Np=2, Nu=2, tol=1e-4)))
    for nb, workers in ((3, 1), (9, 2)):
        other = quiet(cn.solve, cn.preset_spec("example1", **dict(FAST, Np=2, Nu=2, tol=1e-4)),
                      plan=cn.partition(9, nb), workers=workers)
        assert other.iterations == base.iterations
        assert np.array_equal(other.values.values, base.values.values)
        assert np.array_equal(other.policy.values, base.policy.values)
    again = quiet(cn.solve, cn.preset_spec("example1", **dict(FAST, Np=2, Nu=2, tol=1e-4)),
                  init=(base.values, base.policy))
    assert again.converged and again.iterations <= 2
    with pytest.raises(ValueError):  # a plan must cover the grid exactly
        cn.solve(cn.preset_spec("example1", **dict(FAST, Np=2, Nu=2)), plan=cn.BlockPlan(2, 4))


def test_three_player_chain_symmetry(cuda):
    spec = cn.preset_spec("example3", rho=0.5, h=0.01, P_max=0.5, U_max=0.5, tol=1e-8, Np=2, Nu=2,
                          max_iters=20_000)
    res = quiet(cn.solve, spec)
    assert res.converged
    u0 = res.policy.values[0].reshape(3, 3, 3, order="F")
    u2 = res.policy.values[2].reshape(3, 3, 3, order="F")
    np.testing.assert_allclose(u0, u2.transpose(2, 1, 0), atol=1e-8)


def test_fit_policy_and_simulate_vs_reference(cuda):
    spec = spec_of("e1b")
    grid = cn.build_state_grid(spec)
    pol = cn.PolicyField(GOLD["e1b_solve_policy"])
    pols = cn.fit_policy(grid, pol)
    np.testing.assert_allclose(np.stack([p.coefficients for p in pols]), GOLD["e1b_fitpolicy"], rtol=RTOL, atol=ATOL)
    path = cn.simulate(spec, pols, GOLD["e1b_sim_p0"], 500)
    np.testing.assert_allclose(path.states, GOLD["e1b_sim_states"], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(path.controls, GOLD["e1b_sim_controls"], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(cn.discounted_payoff(spec, path.states, path.controls, 400), GOLD["e1b_sim_payoff"],
                               rtol=RTOL, atol=1e-13)


def test_nonfinite_initial_values_rejected(cuda):
    spec = cn.preset_spec("example1", **dict(FAST, Np=2, Nu=2))
    v = np.zeros((2, 9))
    v[0, 3] = np.nan
    with pytest.raises(ValueError, match="finite"):
        cn.solve(spec, init=(v, np.full((2, 9), 0.25)))
    with pytest.raises(ValueError):
        cn.solve(spec, init=(np.zeros((2, 9)), np.full((2, 9), 0.75)))


def test_simulate_batch_matches_single(cuda):
    spec = spec_of("e1b")
    grid = cn.build_state_grid(spec)
    pols = cn.fit_policy(grid, cn.PolicyField(GOLD["e1b_solve_policy"]))
    P0 = np.array([[0.05, 0.3], [0.0, 0.0], [0.5, 0.5], [0.2, 0.1]])
    S, U = cn.simulate_batch(spec, pols, P0, 300)
    for b in range(P0.shape[0]):
        path = cn.simulate(spec, pols, P0[b], 300)
        assert np.array_equal(path.states, S[b]) and np.array_equal(path.controls, U[b])
    with pytest.raises(ValueError):
        cn.simulate(spec, pols, [0.6, 0.1], 10)
    with pytest.raises(ValueError):
        cn.simulate(spec, pols[:1], [0.1, 0.1], 10)


def test_acceptance_value_consistency_and_symmetry(cuda):
    """T/test_acceptance.py #9 (converged example1 values match truncated simulated payoffs from 10
    nodes, horizon log(1e-8)/log(delta)) and #7 (player-exchange symmetries of the simulated
    controls for example3 / example4), with the rollouts batched in one kernel."""
    spec = cn.preset_spec("example1", tol=1e-8)
    res = quiet(cn.solve, spec)
    assert res.converged
    grid = cn.build_state_grid(spec)
    pols = cn.fit_policy(grid, res.policy)
    horizon = int(np.ceil(np.log(1e-8) / np.log(spec.delta)))
    nodes = np.random.default_rng(20240801 + 4).choice(grid.n_nodes, size=10, replace=False)
    S, U = cn.simulate_batch(spec, pols, grid.nodes[nodes], horizon)
    worst = 0.0
    for k, j in enumerate(nodes):
        pay = cn.discounted_payoff(spec, S[k], U[k], horizon)
        worst = max(worst, float(np.max(np.abs(pay - res.values.values[:, j]))))
    assert worst < max(1e-3, 10 * spec.tol)
    for preset, (i, j) in {"example3": (0, 2), "example4": (2, 3)}.items():
        sp = cn.preset_spec(preset)
        r = quiet(cn.solve, sp)
        assert r.converged
        path = cn.simulate(sp, cn.fit_policy(cn.build_state_grid(sp), r.policy), np.zeros(sp.J), 10_000)
        np.testing.assert_allclose(path.controls[:, i], path.controls[:, j], atol=1e-6)


def test_acceptance_plan_invariance_512_nodes(cuda):
    """T/test_acceptance.py #8: example3 at degree 7 (512 nodes), plans 1/8/64/256 blocks and 1/2
    workers give bitwise-identical values, policies and histories."""
    spec = cn.preset_spec("example3", Np=7, Nu=7, h=1e-2, tol=1e-3, max_iters=20_000)
    n = int(np.prod(spec.Np + 1))
    assert n == 512
    base = quiet(cn.solve, spec, plan=cn.partition(n, 1), workers=1)
    assert base.converged
    for nb, workers in ((8, 1), (64, 1), (256, 1), (8, 2), (64, 2)):
        other = quiet(cn.solve, spec, plan=cn.partition(n, nb), workers=workers)
        assert other.converged and other.iterations == base.iterations
        assert np.array_equal(other.values.values, base.values.values)
        assert np.array_equal(other.policy.values, base.policy.values)
        assert np.array_equal(other.history, base.history)
