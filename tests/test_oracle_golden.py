"""CPU: pin the oracle (oracle/cheb_oracle.py) to the reference.

(1) Golden fixtures produced by the reference itself (tests/golden/make_golden.py).
(2) The reference test suite's own known answers for this path (T/test_cheb1d.py,
    T/test_chebnd.py, T/test_acceptance.py criteria 1-3), re-run against the oracle.
"""

import os

import numpy as np
import pytest

from oracle import cheb_oracle as orc

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
RTOL, ATOL = 1e-12, 1e-11


def close(a, b, rtol=RTOL, atol=ATOL):
    np.testing.assert_allclose(np.asarray(a), np.asarray(b), rtol=rtol, atol=atol)


@pytest.mark.parametrize("n", range(0, 65))
def test_transform_1d_vs_reference(n):
    close(orc.cheb_transform(GOLD[f"t1d_in_{n}"]), GOLD[f"t1d_out_{n}"], rtol=0, atol=1e-15)


def test_transform_axes_vs_reference():
    for ax in range(3):
        close(orc.cheb_transform(GOLD["taxis_in"], axis=ax), GOLD[f"taxis_out_{ax}"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("key", ["c1", "c2", "c3", "c4", "c5", "r0", "r1", "r2", "r3", "r4", "r5"])
def test_build_and_eval_vs_reference(key):
    C = orc.tensor_coeffs(GOLD[f"{key}_values"])
    assert np.array_equal(C, GOLD[f"{key}_coef"])  # same numpy ops -> bitwise
    close(orc.eval_points(C, GOLD[f"{key}_points"]), GOLD[f"{key}_eval"], rtol=0, atol=1e-14)
    if f"{key}_evalfull" in GOLD:
        got = [orc.eval_full(C, p) for p in GOLD[f"{key}_points"][:8]]
        close(got, GOLD[f"{key}_evalfull"])


def test_axis_stack_gather_vs_reference():
    close(orc.eval_axis(GOLD["axis_coef"], GOLD["axis_points"]), GOLD["axis_out"], rtol=0, atol=1e-15)
    close(orc.eval_axis_stack(GOLD["stack_coef"], GOLD["stack_points"]), GOLD["stack_axis"], rtol=0, atol=1e-15)
    close(orc.eval_diagonal(GOLD["stack_coef"], GOLD["stack_points"]), GOLD["stack_diag"], rtol=0, atol=1e-15)
    assert np.array_equal(orc.gather_index(GOLD["stack_coef"].shape[:-1], 6), GOLD["stack_gather_flat"])
    close(orc.stack_coeffs(GOLD["stackc_in"]), GOLD["stackc_out"], rtol=0, atol=1e-15)
    close(orc.row_basis(GOLD["basis_points"], 7), GOLD["basis_out"], rtol=0, atol=0)
    targets = [GOLD[f"grid_t{j}"] for j in range(3)]
    close(orc.eval_grid(GOLD["axis_coef"], targets), GOLD["grid_out"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("key", ["loopa", "loopb", "loopc"])
def test_advect_loop_vs_reference(key):
    V = orc.advect_loop(GOLD[f"{key}_V0"], GOLD[f"{key}_A"], 0.01, int(GOLD[f"{key}_steps"]))
    close(V, GOLD[f"{key}_V"], rtol=0, atol=1e-13)


def test_config3_two_steps_vs_reference():
    from paper_2307_04688_b200 import workloads

    w = workloads.make("3", steps=2)
    V = orc.advect_loop(w.values, w.A, w.dt, 2)
    close(V.ravel()[GOLD["c3full_idx"]], GOLD["c3full_V2_sample"], rtol=0, atol=1e-13)
    assert abs(V.sum() - float(GOLD["c3full_V2_sum"])) < 1e-9


# ---- the reference tests' known answers, against the oracle -------------------------------------

def test_direct_sum_all_degrees():
    # T/test_cheb1d.py:253-259 (seed 23) and T/test_acceptance.py:81-96
    rng = np.random.default_rng(23)
    for n in range(1, 65):
        s = rng.standard_normal(n + 1)
        np.testing.assert_allclose(orc.cheb_transform(s), orc.direct_transform(s), atol=1e-12)


def test_constant_and_identity():
    # T/test_cheb1d.py:90-102
    for n in (1, 2, 5, 8):
        e = np.zeros(n + 1)
        e[0] = 1.0
        np.testing.assert_allclose(orc.cheb_transform(np.ones(n + 1)), e, atol=1e-15)
    np.testing.assert_allclose(orc.cheb_transform([1.0, 0.0, -1.0]), [0.0, 1.0, 0.0], atol=1e-15)


def test_tensor_known_answers():
    # T/test_chebnd.py:47-72: constant surface, x*y -> T1 (x) T1, separable outer product
    C = orc.tensor_coeffs(np.ones((4, 3)))
    e = np.zeros((4, 3))
    e[0, 0] = 1.0
    np.testing.assert_allclose(C, e, atol=1e-15)
    nodes = orc.reference_nodes(2)
    X, Y = np.meshgrid(nodes, nodes, indexing="ij")
    e = np.zeros((3, 3))
    e[1, 1] = 1.0
    np.testing.assert_allclose(orc.tensor_coeffs(X * Y), e, atol=1e-15)
    rng = np.random.default_rng(31)
    fx, gy = rng.standard_normal(6), rng.standard_normal(8)
    np.testing.assert_allclose(orc.tensor_coeffs(np.outer(fx, gy)),
                               np.outer(orc.cheb_transform(fx), orc.cheb_transform(gy)), atol=1e-12)


def test_acceptance_criterion_1_exactness():
    # T/test_acceptance.py:50-74 (seed RNG_SEED): polynomials of the basis degrees are exact
    rng = np.random.default_rng(20240801)
    letters = "abcd"
    for _ in range(12):
        n = int(rng.integers(1, 5))
        degrees = rng.integers(1, 7, size=n)
        mono = rng.standard_normal(tuple(degrees + 1))
        nodes = [orc.reference_nodes(int(d)) for d in degrees]
        grids = np.meshgrid(*nodes, indexing="ij")
        vander = [g[..., None] ** np.arange(degrees[d] + 1) for d, g in enumerate(grids)]
        sub_in = ",".join(f"...{letters[d]}" for d in range(n))
        samples = np.einsum(f"{letters[:n]},{sub_in}->...", mono, *vander)
        C = orc.tensor_coeffs(samples)
        pts = rng.uniform(-1.0, 1.0, (100, n))
        van_p = [pts[:, d, None] ** np.arange(degrees[d] + 1) for d in range(n)]
        sub_p = ",".join(f"p{letters[d]}" for d in range(n))
        expect = np.einsum(f"{letters[:n]},{sub_p}->p", mono, *van_p)
        np.testing.assert_allclose(orc.eval_points(C, pts), expect, atol=1e-10)


def test_clamp_semantics():
    # S/cheb1d.py:127-135; T/test_cheb1d.py:161-165
    assert orc.clamp_reference(1.0 + 1e-13) == 1.0
    with pytest.raises(ValueError, match="beyond tolerance"):
        orc.clamp_reference([0.0, 1.0 + 1e-9])
    with pytest.raises(ValueError, match="finite"):
        orc.clamp_reference([np.nan])
