"""GPU: the CUDA path against the reference's own outputs (tests/golden/golden_v1.npz, produced by
tests/golden/make_golden.py from chebnash itself).  fp64 tolerance: allclose(rtol=1e-12,
atol=1e-11) (BASELINE.json north star); index work (gather) exact."""

import os

import numpy as np
import pytest

import paper_2307_04688_b200 as cn

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
RTOL, ATOL = 1e-12, 1e-11


def close(a, b, rtol=RTOL, atol=ATOL):
    np.testing.assert_allclose(np.asarray(a), np.asarray(b), rtol=rtol, atol=atol)


def test_transform_1d(cuda):
    for n in range(0, 65):
        c = cn.coeffs_from_samples(GOLD[f"t1d_in_{n}"], cn.make_basis(n, -1.0, 1.0)).coefficients
        close(c, GOLD[f"t1d_out_{n}"], rtol=0, atol=1e-13)
    for ax in range(3):
        close(cn.cheb_transform(GOLD["taxis_in"], axis=ax), GOLD[f"taxis_out_{ax}"])


@pytest.mark.parametrize("key,lo", [("c1", 0.0), ("c2", 0.0), ("c3", 0.0), ("c4", 0.0), ("c5", 0.0), ("r0", -1.0),
                                    ("r1", -1.0), ("r2", -1.0), ("r3", -1.0), ("r4", -1.0), ("r5", -1.0)])
def test_build_and_eval(cuda, key, lo):
    vals = GOLD[f"{key}_values"]
    bases = [cn.make_basis(n - 1, lo, 1.0) for n in vals.shape]
    t = cn.tensor_coeffs(vals, bases)
    close(t.coefficients, GOLD[f"{key}_coef"])
    close(cn.eval_points(t, GOLD[f"{key}_points"]), GOLD[f"{key}_eval"])
    if f"{key}_evalfull" in GOLD:
        got = [cn.eval_full(t, p) for p in GOLD[f"{key}_points"][:8]]
        close(got, GOLD[f"{key}_evalfull"])


def test_axis_stack_gather(cuda):
    tc = GOLD["axis_coef"]
    t = cn.CoefTensor([cn.make_basis(n - 1, -1.0, 1.0) for n in tc.shape], tc)
    close(cn.eval_axis(t, GOLD["axis_points"]), GOLD["axis_out"])
    sc = GOLD["stack_coef"]
    st = cn.TensorStack([cn.make_basis(n - 1, -1.0, 1.0) for n in sc.shape[:-1]], sc)
    close(cn.eval_axis(st, GOLD["stack_points"]), GOLD["stack_axis"])
    g = cn.make_gather_index(sc.shape[:-1], 6)
    assert np.array_equal(g.flat, GOLD["stack_gather_flat"])
    close(cn.eval_diagonal_batch(st, GOLD["stack_points"], g).coefficients, GOLD["stack_diag"])
    close(g.take(cn.eval_axis(st, GOLD["stack_points"])), GOLD["stack_gather_take"])
    close(cn.stack_coeffs(GOLD["stackc_in"], [cn.make_basis(3, -1, 1), cn.make_basis(4, -1, 1)]).coefficients,
          GOLD["stackc_out"])
    close(cn.basis_matrix(GOLD["basis_points"], 6), GOLD["basis_out"], rtol=0, atol=1e-14)
    targets = [GOLD[f"grid_t{j}"] for j in range(3)]
    close(cn.eval_grid(t, targets), GOLD["grid_out"])


@pytest.mark.parametrize("key", ["loopa", "loopb", "loopc"])
def test_advect_loop(cuda, key):
    V0 = GOLD[f"{key}_V0"]
    bases = [cn.make_basis(n - 1, 0.0, 1.0) for n in V0.shape]
    V = cn.advect_loop(V0, bases, GOLD[f"{key}_A"], 0.01, int(GOLD[f"{key}_steps"]))
    close(V, GOLD[f"{key}_V"])


def test_config3_two_steps(cuda):
    from paper_2307_04688_b200 import workloads

    w = workloads.make("3", steps=2)
    bases = [cn.make_basis(w.n - 1, 0.0, 1.0)] * w.J
    V = cn.advect_loop(w.values, bases, w.A, w.dt, 2)
    close(V.ravel()[GOLD["c3full_idx"]], GOLD["c3full_V2_sample"])
    assert abs(V.sum() - float(GOLD["c3full_V2_sum"])) < 1e-8
