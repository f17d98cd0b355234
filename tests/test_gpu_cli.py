"""GPU: the closed-form LQ oracle on the device (cb_lq) against the reference's own outputs, and the
command-line front end end to end (the reference's T/test_cli.py behaviours and formats;
SURVEY.md §8f row 4)."""

import json
import os
import warnings

import numpy as np
import pytest

import paper_2307_04688_b200 as cn
from paper_2307_04688_b200.cli import main
from oracle import solver_oracle as so

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_solver_v1.npz"))
FAST = ["--h", "0.01", "--tol", "1e-4", "--rho", "0.5", "--np", "2", "--nu", "2"]


def spec_of(key):
    g = so.game_from_golden(GOLD, key)
    return cn.GameSpec(J=g.J, K=g.K, beta=g.beta, phi=g.phi, A=g.A, c=g.c, m=g.m, rho=g.rho, h=g.h, P_max=g.P_max,
                       U_max=g.U_max, Np=g.Np, Nu=g.Nu, tol=g.tol, max_iters=g.max_iters)


def quiet_main(args):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return main(args)


def read_csv(path):
    return np.genfromtxt(path, delimiter=",", names=True)


@pytest.mark.parametrize("key", ["lq1", "lq2", "lq3", "lq4"])
def test_lq_solve_and_update_vs_reference(cuda, key):
    spec = spec_of(key)
    fb = cn.lq_solve(spec)
    for name in ("Q", "b", "d", "e", "f"):
        np.testing.assert_allclose(getattr(fb, name), GOLD[f"{key}_{name}"], rtol=1e-10, atol=1e-12)
    assert abs(fb.iterations - int(GOLD[f"{key}_iterations"])) <= 1
    assert fb.negative_fraction == float(GOLD[f"{key}_negfrac"])
    assert fb.high_fraction == float(GOLD[f"{key}_highfrac"])
    upd = cn.lq_bellman_update(spec, *[GOLD[f"{key}_upd_in_{n}"] for n in ("Q", "b", "d", "e", "f")])
    for name, got in zip(("Q", "b", "d", "e", "f"), upd):
        np.testing.assert_allclose(got, GOLD[f"{key}_upd_out_{name}"], rtol=1e-13, atol=1e-15)


def test_policy_error_vs_reference(cuda):
    spec = spec_of("e1b")
    grid = cn.build_state_grid(spec)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        res = cn.solve(spec)
    err = cn.policy_error(res.policy, cn.lq_solve(spec, grid), grid)
    assert abs(err - float(GOLD["perr_e1b"])) <= 1e-9 * max(1.0, abs(float(GOLD["perr_e1b"])))


def test_acceptance_oracle_envelope(cuda):
    """T/test_acceptance.py #6: the policy error against the closed form decreases over degrees 2/4/8."""
    errors = {}
    for degree in (2, 4, 8):
        spec = cn.preset_spec("example1", Np=degree, Nu=degree)
        grid = cn.build_state_grid(spec)
        fb = cn.lq_solve(spec, grid)
        assert fb.negative_fraction == 0.0
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            res = cn.solve(spec)
        assert res.converged
        errors[degree] = cn.policy_error(res.policy, fb, grid)
    assert errors[2] > errors[4] > errors[8] and errors[8] < 1e-2


def test_cli_solve_outputs_and_rerun_bitwise(cuda, tmp_path):
    out = tmp_path / "run"
    assert quiet_main(["solve", "--preset", "example1", *FAST, "--out", str(out)]) == 0
    policy = read_csv(out / "policy.csv")
    assert policy.dtype.names == ("node", "p_1", "p_2", "u_1", "u_2") and policy.shape[0] == 9
    assert read_csv(out / "value.csv").dtype.names == ("node", "p_1", "p_2", "V_1", "V_2")
    conv = read_csv(out / "convergence.csv")
    assert conv.dtype.names == ("iteration", "supdiff_1", "supdiff_2") and conv["supdiff_1"][-1] < 1e-4
    cfg = json.loads((out / "run.json").read_text())
    assert cfg["schema_version"] == 1 and cfg["preset"] == "example1"
    assert cfg["game"]["h"] == 0.01 and cfg["game"]["Np"] == [2, 2] and cfg["game"]["K"] == [[-1.0, 1.0], [1.0, -1.0]]
    text = (out / "policy.csv").read_bytes()
    assert b"\r" not in text and b"e-" in text or b"e+" in text
    # re-run from the written run.json reproduces every output bitwise
    out2 = tmp_path / "again"
    assert quiet_main(["solve", "--config", str(out / "run.json"), "--out", str(out2)]) == 0
    for name in ("policy.csv", "value.csv", "convergence.csv"):
        assert (out / name).read_bytes() == (out2 / name).read_bytes()
    # the CSV policy is the library's policy, losslessly
    spec = cn.preset_spec("example1", h=0.01, tol=1e-4, rho=0.5, Np=2, Nu=2)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = cn.solve(spec)
    for i in range(2):
        np.testing.assert_array_equal(policy[f"u_{i+1}"], res.policy.values[i])


def test_cli_presets_nonconvergence_and_simulate(cuda, tmp_path):
    out3 = tmp_path / "e3"
    assert quiet_main(["solve", "--preset", "example3", *FAST, "--out", str(out3)]) == 0
    assert json.loads((out3 / "run.json").read_text())["game"]["K"][1] == [1.0, -2.0, 1.0]
    rc = quiet_main(["solve", "--preset", "example1", "--h", "0.01", "--rho", "0.5", "--np", "2", "--nu", "2",
                     "--tol", "1e-14", "--out", str(tmp_path / "nc"), "--config", str(_cfg(tmp_path, 5))])
    assert rc == 3
    out = tmp_path / "run"
    quiet_main(["solve", "--preset", "example1", *FAST, "--out", str(out)])
    assert main(["simulate", "--out", str(out), "--sim-horizon", "2.0", "--p0", "0,0"]) == 0
    path = read_csv(out / "timepath.csv")
    assert path.dtype.names == ("t", "p_1", "p_2", "u_1", "u_2") and path.shape[0] == 201
    np.testing.assert_allclose(path["u_1"], path["u_2"], atol=1e-6)
    assert main(["simulate", "--out", str(out), "--sim-horizon", "0", "--p0", "0.1,0.2"]) == 0
    rows = (out / "timepath.csv").read_text().strip().split("\n")
    assert len(rows) == 2 and float(rows[1].split(",")[1]) == pytest.approx(0.1)


def _cfg(tmp_path, max_iters):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps({"game": {"max_iters": max_iters}}))
    return p


def test_cli_compare_and_bench_blocks(cuda, tmp_path, capsys):
    args = ["compare", "--preset", "example1", "--h", "0.01", "--tol", "1e-4", "--rho", "0.5", "--np-list", "2,4"]
    out1, out2 = tmp_path / "a", tmp_path / "b"
    assert quiet_main([*args, "--out", str(out1)]) == 0
    table = read_csv(out1 / "error.csv")
    assert tuple(table.dtype.names) == ("np", "error", "wall_time") and table["error"][0] > table["error"][1]
    assert quiet_main([*args, "--out", str(out2)]) == 0
    col = lambda o: [ln.split(",")[1] for ln in (o / "error.csv").read_text().splitlines()[1:]]  # noqa: E731
    assert col(out1) == col(out2)
    capsys.readouterr()
    out = tmp_path / "bb"
    assert quiet_main(["bench-blocks", "--preset", "example1", "--h", "0.01", "--tol", "1e-3", "--rho", "0.5",
                       "--np", "2", "--nu", "2", "--reps", "1", "--out", str(out)]) == 0
    bt = read_csv(out / "blocks.csv")
    np.testing.assert_array_equal(bt["n_b"], [1, 3, 9])
    np.testing.assert_array_equal(bt["n_b"] * bt["n_f"], [9, 9, 9])
    sweeps = {ln.split("(")[1] for ln in capsys.readouterr().out.splitlines() if "sweeps" in ln}
    assert len(sweeps) == 1
