"""CPU: the solver restatement (oracle/solver_oracle.py) against the reference solver's own outputs
(tests/golden/golden_solver_v1.npz from tests/golden/make_golden_solver.py), plus the host-side
solver plumbing of the product (plans, GameSpec validation, presets).  No kernel runs here."""

import os

import numpy as np
import pytest

from oracle import solver_oracle as so

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_solver_v1.npz"))
KEYS = ["e1a", "e1b", "e1c", "e3a", "e4a", "e1d"]


@pytest.mark.parametrize("key", KEYS)
def test_oracle_sweep_and_stacks_match_reference(key):
    game = so.game_from_golden(GOLD, key)
    S = so.Solver(game)
    for i in range(game.J):
        np.testing.assert_allclose(S.stacks[i], GOLD[f"{key}_stack{i}"], rtol=0, atol=1e-15)
    u1, v1, _ = S.sweep(S.refit(GOLD[f"{key}_sweep_v0"]), GOLD[f"{key}_sweep_u0"])
    np.testing.assert_allclose(v1, GOLD[f"{key}_sweep_v1"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(u1, GOLD[f"{key}_sweep_u1"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("key", ["e1d", "e4a"])
def test_oracle_solve_matches_reference(key):
    game = so.game_from_golden(GOLD, key)
    r = so.Solver(game).solve()
    assert r["iterations"] == int(GOLD[f"{key}_solve_iterations"])
    assert r["converged"] == bool(GOLD[f"{key}_solve_converged"])
    np.testing.assert_allclose(r["values"], GOLD[f"{key}_solve_values"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(r["policy"], GOLD[f"{key}_solve_policy"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(r["history"], GOLD[f"{key}_solve_history"], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("L", [2, 3, 5, 9])
def test_oracle_maximiser_bitwise(L):
    x, f = so.maximise_rows(GOLD[f"maxblock{L}_coef"], GOLD[f"maxblock{L}_x0"])
    assert np.array_equal(x, GOLD[f"maxblock{L}_x"]) and np.array_equal(f, GOLD[f"maxblock{L}_f"])


def test_oracle_newton_maximize_bitwise():
    got = [so.newton_maximize(r, 0.0, 1.0, u0) for r, u0 in zip(GOLD["newton_rows"], GOLD["newton_u0"])]
    assert np.array_equal([g[0] for g in got], GOLD["newton_u"])
    assert np.array_equal([g[1] for g in got], GOLD["newton_f"])


def test_oracle_simulate_matches_reference():
    game = so.game_from_golden(GOLD, "e1b")
    pols = list(GOLD["e1b_fitpolicy"])
    states, controls = so.simulate(game, pols, GOLD["e1b_sim_p0"], 500)
    np.testing.assert_allclose(states, GOLD["e1b_sim_states"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(controls, GOLD["e1b_sim_controls"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(so.discounted_payoff(game, states, controls, 400), GOLD["e1b_sim_payoff"],
                               rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------------------------------------
# host-side plumbing of the product (no GPU needed)
# ---------------------------------------------------------------------------------------------

def test_partition_semantics():
    import paper_2307_04688_b200 as cn

    assert cn.partition(512, 1).slices() == [slice(0, 512)]
    assert len(cn.partition(512, 512).slices()) == 512
    seen = np.zeros(512, dtype=int)
    for sl in cn.partition(512, 8).slices():
        seen[sl] += 1
    assert (seen == 1).all()
    with pytest.raises(ValueError):
        cn.partition(512, 7)
    with pytest.raises(ValueError):
        cn.BlockPlan(0, 4)


def test_gamespec_validation_and_presets():
    import paper_2307_04688_b200 as cn

    s = cn.preset_spec("example3")
    assert s.J == 3 and s.delta == 1.0 - 0.1 * 1e-3 and tuple(s.Np) == (3, 3, 3)
    assert cn.spec_to_dict(cn.spec_from_dict(cn.spec_to_dict(s))) == cn.spec_to_dict(s)
    for bad in (dict(J=1), dict(h=20.0), dict(U_max=0.1), dict(phi=-1.0), dict(Np=0), dict(max_iters=0)):
        with pytest.raises(ValueError):
            cn.preset_spec("example1", **bad)
    with pytest.raises(ValueError):
        cn.preset_spec("example2")
    g = cn.build_state_grid(cn.preset_spec("example1", Np=2))
    assert g.shape == (3, 3) and g.n_nodes == 9
    assert np.array_equal(g.nodes[:3, 1], np.full(3, g.nodes[0, 1]))  # dim 1 fastest
    game = so.game_from_golden(GOLD, "e3a")
    np.testing.assert_array_equal(so.grid_nodes(game), cn.build_state_grid(cn.preset_spec(
        "example3", rho=0.5, h=0.01, P_max=0.5, U_max=0.5, tol=1e-8, Np=2, Nu=2)).nodes)


def test_game_struct_matches_header_size():
    import ctypes

    from paper_2307_04688_b200 import _lib

    # int J + 2*int[8] (+4 pad) + 5 doubles + A, phi + K[8][8] + beta, c, m + 2 * double[8][32]
    assert ctypes.sizeof(_lib.CbGame) == 72 + 40 + 128 + 512 + 192 + 4096
