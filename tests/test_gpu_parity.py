"""GPU parity: the CUDA path (through the C ABI / Python shim) against the CPU oracle
(oracle/cheb_oracle.py, pinned to the reference in test_oracle_golden.py) on the same seeded inputs.

Tolerance (north star, BASELINE.json): fp64 allclose with rtol = 1e-12 and atol = 1e-11 — summation
order differs from numpy's pocketfft / OpenBLAS, so pure 1e-12 relative is not meaningful where
|V| is tiny.  Integer / index work (gather indices) is compared exactly.
"""

import numpy as np
import pytest

import paper_2307_04688_b200 as cn
from oracle import cheb_oracle as orc
from paper_2307_04688_b200 import workloads

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-12, 1e-11


def close(got, ref, rtol=RTOL, atol=ATOL):
    np.testing.assert_allclose(np.asarray(got), np.asarray(ref), rtol=rtol, atol=atol)


def bases_for(J, n, a=0.0, b=1.0):
    return [cn.make_basis(n - 1, a, b)] * J


# ------------------------------------------------------------------------------------------------
# K1 build
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", ["1", "2", "3", "4", "5a"])
def test_build_baseline_shapes(cuda, cfg):
    w = workloads.make(cfg, M=16)
    t = cn.tensor_coeffs(w.values, bases_for(w.J, w.n))
    close(t.coefficients, orc.tensor_coeffs(w.values))


@pytest.mark.parametrize("shape", [(1,), (2,), (7,), (34,), (65,), (3, 1), (1, 5), (4, 3), (16, 2), (5, 6, 7),
                                   (2, 2, 2, 2), (3, 4, 5, 6), (8, 9, 10), (33, 33), (2, 3, 2, 3, 2, 3),
                                   (3, 3, 3, 3, 3, 3, 3, 3), (12, 12, 12), (40, 41)])
def test_build_ragged_shapes(cuda, shape):
    rng = np.random.default_rng(abs(hash(shape)) % 2**32)
    s = rng.standard_normal(shape)
    bases = [cn.make_basis(d - 1, -1.0, 1.0) for d in shape]
    close(cn.tensor_coeffs(s, bases).coefficients, orc.tensor_coeffs(s))


def test_transform_matches_direct_sum_all_degrees(cuda):
    rng = np.random.default_rng(23)
    for n in range(1, 65):
        s = rng.standard_normal(n + 1)
        c = cn.coeffs_from_samples(s, cn.make_basis(n, -1.0, 1.0)).coefficients
        np.testing.assert_allclose(c, orc.direct_transform(s), atol=1e-12)


def test_cheb_transform_axis(cuda):
    rng = np.random.default_rng(7)
    block = rng.standard_normal((9, 5, 4))
    for axis in range(3):
        close(cn.cheb_transform(block, axis=axis), orc.cheb_transform(block, axis=axis))


def test_build_rejects_nonfinite(cuda):
    s = np.ones((4, 4))
    s[2, 1] = np.nan
    with pytest.raises(ValueError, match="finite"):
        cn.tensor_coeffs(s, bases_for(2, 4))


def test_stack_coeffs(cuda):
    rng = np.random.default_rng(30)
    bases = (cn.make_basis(3, -1.0, 1.0), cn.make_basis(4, -1.0, 1.0))
    samples = rng.standard_normal((4, 5, 6))
    st = cn.stack_coeffs(samples, bases)
    assert st.count == 6
    close(st.coefficients, orc.stack_coeffs(samples))


# ------------------------------------------------------------------------------------------------
# K2 scattered evaluation
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg,M", [("1", 65536), ("2", 20000), ("3", 4096), ("4", 2048), ("5a", 512)])
def test_eval_points_baseline_shapes(cuda, cfg, M):
    if cfg == "3":
        w = workloads.make("3")
        T, _ = orc.advect_points(w.values.shape, w.A, w.dt)
        pts = T[:M]
    elif cfg == "5a":
        w = workloads.make("5a")
        pts = 2.0 * np.random.default_rng(5).random((M, 6)) - 1.0
    else:
        w = workloads.make(cfg, M=M)
        pts = w.points
    t = cn.tensor_coeffs(w.values, bases_for(w.J, w.n))
    ref_c = orc.tensor_coeffs(w.values)
    got = cn.eval_points(t, pts)
    close(got, orc.eval_points(ref_c, pts))


@pytest.mark.parametrize("shape", [(5,), (17,), (3, 4), (17, 17), (2, 9, 3), (6, 1, 5), (1, 1, 1), (9, 9, 9, 9),
                                   (4, 3, 5, 2, 3), (3, 3, 3, 3, 3, 3), (2, 2, 2, 2, 2, 2, 2, 2), (33, 33, 33),
                                   # row-contraction kernel: K % 8 tails 1, 2, 3 and padded
                                   (17, 17, 18), (20, 15, 19), (16, 17, 12), (64, 5, 9), (120, 3, 33), (7, 6, 7, 41)])
@pytest.mark.parametrize("generic", [False, True])
def test_eval_points_ragged(cuda, shape, generic):
    rng = np.random.default_rng(len(shape) * 100 + sum(shape))
    coef = rng.standard_normal(shape)
    J = len(shape)
    t = cn.CoefTensor([cn.make_basis(d - 1, -1.0, 1.0) for d in shape], coef)
    M = 3000
    pts = rng.uniform(-1.0, 1.0, (M, J))
    pts[:5] = np.sign(pts[:5])  # exact endpoints
    from paper_2307_04688_b200 import _lib
    from paper_2307_04688_b200.chebnd import _eval_points_device

    got = _lib.to_host(_eval_points_device(shape, t.device_coefficients, _lib.to_device(pts), force_generic=generic))
    ref = orc.eval_points(coef, pts)
    scale = max(1.0, float(np.abs(coef).sum()))
    close(got, ref, atol=1e-13 * scale)


# q = 2 layouts by row count: >= 1,536 rows -> 12 warps x 8 x 2 DMMA tiles (Roles code 36, 192-row
# stages), >= 192 rows -> 12 warps x 4 x 2 (code 28, 96-row stages), else the 16-warp 2 x 2 shape.
# The shapes cover NL = 0..6 leading modes and partial last row blocks of every valid-m-tile count.
@pytest.mark.parametrize("shape,code", [
    ((6,) * 8, 36), ((5,) * 7, 36), ((7,) * 6, 36), ((40, 41, 6, 7), 36), ((6,) * 7, 36),
    ((6,) * 6, 28), ((5,) * 6, 28), ((15,) * 4, 28), ((7, 7, 7, 6, 6), 28), ((3, 3, 3, 3, 3, 3, 6, 6), 28),
    ((13,) * 4, 16), ((20, 6, 6), 16), ((5,) * 5, 16)])
def test_eval_points_register_tile_shapes(cuda, shape, code):
    from paper_2307_04688_b200 import _lib
    from paper_2307_04688_b200.chebnd import _eval_points_device

    rng = np.random.default_rng(sum(shape) * 7 + len(shape))
    coef = rng.standard_normal(shape)
    J = len(shape)
    t = cn.CoefTensor([cn.make_basis(d - 1, -1.0, 1.0) for d in shape], coef)
    M = 64 * 3 + 37  # ragged last tile
    pts = rng.uniform(-1.0, 1.0, (M, J))
    pts[:3] = np.sign(pts[:3])
    got = _lib.to_host(_eval_points_device(shape, t.device_coefficients, _lib.to_device(pts)))
    plan = _lib.load().cb_last_eval_plan().decode()
    assert _lib.eval_layout(shape)["q"] == 2
    assert f"NCW={code}>" in plan, plan
    ref = orc.eval_points(coef, pts)
    scale = max(1.0, float(np.abs(coef).sum()))
    close(got, ref, atol=1e-13 * scale)
    # the same points in a different batch split: bitwise identical (shape-only kernel choice)
    a = _lib.to_host(_eval_points_device(shape, t.device_coefficients, _lib.to_device(pts[:100])))
    b = _lib.to_host(_eval_points_device(shape, t.device_coefficients, _lib.to_device(pts[100:])))
    assert np.array_equal(np.concatenate([a, b]), got)


@pytest.mark.parametrize("shape", [(17, 17), (5, 9), (34, 34), (1, 7), (9, 1), (2, 2), (33, 20), (17, 17, 17), (40, 5)])
def test_build_eval_points_bitwise_equals_two_calls(cuda, shape):
    """cb_build_eval_points (one fused launch for small J = 2 tensors) against cb_tensor_coeffs +
    cb_eval_points: coefficients and values bitwise, and both against the oracle."""
    from paper_2307_04688_b200 import _lib
    from paper_2307_04688_b200.chebnd import _eval_points_device, tensor_coeffs_device

    lib = _lib.load()
    rng = np.random.default_rng(sum(shape) + 11 * len(shape))
    vals = rng.standard_normal(shape)
    J = len(shape)
    M = 1000
    pts = rng.uniform(-1.0, 1.0, (M, J))
    pts[:4] = np.sign(pts[:4])
    dv, dp = _lib.to_device(vals), _lib.to_device(pts)
    coef2 = tensor_coeffs_device(dv, shape)
    out2 = _lib.to_host(_eval_points_device(shape, coef2, dp))
    coef1 = _lib.empty((_lib.eval_layout(shape)["elems"],))
    coef1.fill_(float("nan"))
    out1 = _lib.empty((M,))
    st = _lib.new_status()
    _lib.check(lib.cb_build_eval_points(J, _lib.i64_array(shape), _lib.ptr(dv), M, _lib.ptr(dp), _lib.ptr(out1),
                                        _lib.ptr(coef1), _lib.ptr(st), _lib.stream_handle()), "build_eval")
    plan = lib.cb_last_eval_plan().decode()
    L = _lib.eval_layout(shape)
    fused = J == 2 and max(shape) <= 34 and L["R"] * L["K"] < 0.75 * L["R8"] * L["Kp"]
    assert plan.startswith("build_eval_j2_kernel") == fused, plan
    assert np.array_equal(_lib.to_host(coef1), _lib.to_host(coef2))
    assert np.array_equal(_lib.to_host(out1), out2)
    close(out2, orc.eval_points(orc.tensor_coeffs(vals), pts))


def test_build_eval_points_reports_nonfinite_samples(cuda):
    from paper_2307_04688_b200 import _lib

    lib = _lib.load()
    vals = np.ones((6, 6))
    vals[3, 2] = np.inf
    pts = np.zeros((8, 2))
    st = _lib.new_status()
    coef = _lib.empty((_lib.eval_layout((6, 6))["elems"],))
    out = _lib.empty((8,))
    _lib.check(lib.cb_build_eval_points(2, _lib.i64_array((6, 6)), _lib.ptr(_lib.to_device(vals)), 8,
                                        _lib.ptr(_lib.to_device(pts)), _lib.ptr(out), _lib.ptr(coef), _lib.ptr(st),
                                        _lib.stream_handle()), "build_eval")
    with pytest.raises(ValueError, match="finite"):
        _lib.raise_for_samples(st)


def test_eval_points_matches_eval_full(cuda):
    rng = np.random.default_rng(43)
    coef = rng.standard_normal((4, 5, 3))
    t = cn.CoefTensor([cn.make_basis(d - 1, -1.0, 1.0) for d in coef.shape], coef)
    pts = rng.uniform(-1, 1, (20, 3))
    got = cn.eval_points(t, pts)
    for i in range(20):
        assert got[i] == pytest.approx(orc.eval_full(coef, pts[i]), abs=1e-12)
        assert cn.eval_full(t, pts[i]) == pytest.approx(orc.eval_full(coef, pts[i]), abs=1e-12)


def test_eval_points_clamp_semantics(cuda):
    t = cn.CoefTensor([cn.make_basis(1, -1.0, 1.0)] * 2, np.array([[1.0, 2.0], [3.0, 4.0]]))
    ok = cn.eval_points(t, np.array([[1.0 + 1e-13, -1.0 - 5e-13]]))
    close(ok, [orc.eval_full(t.coefficients, [1.0, -1.0])])
    with pytest.raises(ValueError, match="beyond tolerance"):
        cn.eval_points(t, np.array([[0.0, 1.0 + 1e-9]]))
    with pytest.raises(ValueError, match="finite"):
        cn.eval_points(t, np.array([[np.nan, 0.0]]))
    with pytest.raises(ValueError):
        cn.eval_full(t, [0.1, 0.2, 0.3])


def test_eval_points_shard_bitwise_invariance(cuda):
    """Any contiguous sub-batch gives bit-identical values (multi-GPU point sharding contract)."""
    w = workloads.make("2", M=8192)
    t = cn.tensor_coeffs(w.values, bases_for(w.J, w.n))
    full = cn.eval_points(t, w.points)
    for a, b in ((0, 4096), (4096, 8192), (17, 3000), (8000, 8192)):
        part = cn.eval_points(t, w.points[a:b])
        assert np.array_equal(part, full[a:b]), (a, b, float(np.abs(part - full[a:b]).max()))


@pytest.mark.parametrize("cfg,M", [("2", 0), ("2", 1000), ("2", 600_000), ("4", 2_100_000), ("3", 300_007)])
def test_eval_points_pinned_host_pipeline(cuda, cfg, M):
    """Pinned host points go through cb_eval_points_host (chunked H2D / eval / D2H on copy
    streams): bit-identical to the device-resident call, result in pinned host memory."""
    import torch

    if cfg == "3":
        w = workloads.make("3")
        points = 2.0 * np.random.default_rng(3).random((M, w.J)) - 1.0
    else:
        w = workloads.make(cfg, M=max(M, 1))
        points = w.points[:M]
    t = cn.tensor_coeffs(w.values, bases_for(w.J, w.n))
    pts = torch.from_numpy(np.ascontiguousarray(points)).pin_memory()
    got = cn.eval_points(t, pts)
    assert isinstance(got, torch.Tensor) and not got.is_cuda and got.shape == (M,)
    assert got.is_pinned() or M == 0  # (an empty tensor reports unpinned)
    ref = cn.eval_points(t, pts.cuda()).cpu()
    assert torch.equal(got, ref)
    if M and M <= 1000:
        close(got.numpy(), orc.eval_points(orc.tensor_coeffs(w.values), points))
    if M:
        bad = pts.clone().pin_memory()
        bad[M // 2, 0] = 1.5
        with pytest.raises(ValueError, match="beyond tolerance"):
            cn.eval_points(t, bad)


def test_polynomial_exactness(cuda):
    # T/test_chebnd.py:355-368 (seed 46): exact for polynomials of the basis degrees
    rng = np.random.default_rng(46)
    degrees = (3, 2, 4)
    bases = tuple(cn.make_basis(n, -1.0, 1.0) for n in degrees)
    mono = rng.standard_normal(tuple(d + 1 for d in degrees))
    grids = np.meshgrid(*(b.nodes for b in bases), indexing="ij")
    samples = np.polynomial.polynomial.polyval3d(*grids, mono)
    t = cn.tensor_coeffs(samples, bases)
    pts = rng.uniform(-1, 1, (100, 3))
    close(cn.eval_points(t, pts), np.polynomial.polynomial.polyval3d(*pts.T, mono), rtol=0, atol=1e-10)


# ------------------------------------------------------------------------------------------------
# axis / stack / gather API
# ------------------------------------------------------------------------------------------------

def test_eval_axis_tensor_and_stack(cuda):
    rng = np.random.default_rng(35)
    coef = rng.standard_normal((5, 4, 3))
    t = cn.CoefTensor([cn.make_basis(d - 1, -1.0, 1.0) for d in coef.shape], coef)
    pts = rng.uniform(-1, 1, 7)
    close(cn.eval_axis(t, pts), orc.eval_axis(coef, pts))
    sc = rng.standard_normal((4, 3, 6))
    st = cn.TensorStack([cn.make_basis(3, -1, 1), cn.make_basis(2, -1, 1)], sc)
    close(cn.eval_axis(st, pts), orc.eval_axis_stack(sc, pts))
    with pytest.raises(ValueError):
        cn.eval_axis(t, [])
    with pytest.raises(ValueError):
        cn.eval_axis(t, [1.5])


def test_diagonal_batch_and_gather(cuda):
    rng = np.random.default_rng(39)
    sc = rng.standard_normal((5, 3, 4, 6))
    bases = [cn.make_basis(d - 1, -1, 1) for d in sc.shape[:-1]]
    st = cn.TensorStack(bases, sc)
    pts = rng.uniform(-1, 1, 6)
    g = cn.make_gather_index(sc.shape[:-1], 6)
    assert np.array_equal(g.flat, orc.gather_index(sc.shape[:-1], 6))
    direct = cn.eval_diagonal_batch(st, pts, g)
    close(direct.coefficients, orc.eval_diagonal(sc, pts))
    gathered = g.take(cn.eval_axis(st, pts))
    close(gathered, direct.coefficients)
    with pytest.raises(ValueError):
        cn.eval_diagonal_batch(st, np.zeros(5), g)
    with pytest.raises(ValueError):
        cn.eval_diagonal_batch(st, pts, cn.make_gather_index((99, 2), 6))


def test_full_binding_chain_matches_naive(cuda):
    # T/test_chebnd.py:588-600 pattern (batched = naive), seed 44
    rng = np.random.default_rng(44)
    for _ in range(10):
        ndim = int(rng.integers(1, 5))
        count = int(rng.integers(1, 33))
        bases = tuple(cn.make_basis(int(rng.integers(1, 7)), -1.0, 1.0) for _ in range(ndim))
        sc = rng.standard_normal(tuple(b.size for b in bases) + (count,))
        pts = rng.uniform(-1.0, 1.0, (ndim, count))
        cur = cn.TensorStack(bases, sc)
        for d in range(ndim):
            g = cn.make_gather_index(cur.coefficients.shape[:-1], count)
            cur = cn.eval_diagonal_batch(cur, pts[d], g)
        naive = np.array([orc.eval_full(sc[..., j], pts[:, j]) for j in range(count)])
        np.testing.assert_allclose(cur.coefficients, naive, atol=1e-11)


def test_basis_matrix_and_private_kernels(cuda):
    pts = np.linspace(-1, 1, 9)
    close(cn.basis_matrix(pts, 6), np.cos(np.arange(7)[None, :] * np.arccos(pts)[:, None]), rtol=0, atol=1e-13)
    from paper_2307_04688_b200 import chebnd as nd

    rng = np.random.default_rng(3)
    B = rng.standard_normal((5, 4))
    F = rng.standard_normal((4, 7))
    close(nd._bind_rows(B, F), B @ F)
    S = rng.standard_normal((3, 4, 7))
    close(nd._bind_shared(B, S), np.matmul(B, S))
    Bd = rng.standard_normal((3, 4))
    close(nd._bind_diagonal(Bd, S), np.matmul(Bd[:, None, :], S)[:, 0, :])
    close(nd._row_basis(pts, 5), orc.row_basis(pts, 5))


def test_eval_1d_clenshaw_derivative(cuda):
    rng = np.random.default_rng(9)
    coef = rng.standard_normal(10)
    c = cn.CoefVector(coef, cn.make_basis(9, -1.0, 1.0))
    xs = np.linspace(-1, 1, 21)
    close(cn.eval_1d(c, xs), orc.clenshaw(coef, xs))
    assert cn.eval_1d(c, 0.7) == pytest.approx(orc.clenshaw(coef, 0.7), abs=1e-13)
    batch = rng.standard_normal((6, 4, 3))
    xb = rng.uniform(-1, 1, (4, 3))
    close(cn.clenshaw(batch, xb), orc.clenshaw(batch, xb))
    close(cn.derivative_array(batch.transpose(1, 2, 0)), orc.derivative_array(batch.transpose(1, 2, 0)))
    with pytest.raises(ValueError):
        cn.eval_1d(c, 1.0 + 1e-9)


# ------------------------------------------------------------------------------------------------
# K3 structured evaluation, K4 loop
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("shape,k", [((13, 13, 13), (25, 7, 3)), ((5, 4, 3, 6), (2, 3, 4, 5)), ((17,), (40,)),
                                     ((3, 3, 3, 3, 3, 3), (5, 5, 5, 5, 5, 5)), ((5, 5, 5), (4, 4, 4)),
                                     ((13, 13, 13, 13), (25, 25, 25, 25)), ((4, 17, 17), (3, 25, 25)),
                                     # fused last pair: q = 1 (unpadded copy) and q = 2 (padded rows carried)
                                     ((3, 5, 5), (2, 4, 4)), ((2, 13, 13), (3, 25, 25)), ((7, 3, 13, 13), (5, 4, 25, 25)),
                                     ((40, 5, 5), (9, 4, 4)),
                                     # several fused pairs in sequence (config 5a's plan), odd J
                                     ((5, 5, 5, 5, 3), (4, 4, 4, 4, 2)), ((13, 13, 5, 5, 5, 5), (25, 25, 4, 4, 4, 4)),
                                     ((5, 5, 5, 5, 5), (4, 4, 4, 4, 4))])
def test_eval_grid(cuda, shape, k):
    rng = np.random.default_rng(sum(shape))
    coef = rng.standard_normal(shape)
    t = cn.CoefTensor([cn.make_basis(d - 1, -1.0, 1.0) for d in shape], coef)
    targets = [np.linspace(-1, 1, kk) for kk in k]
    close(cn.eval_grid(t, targets), orc.eval_grid(coef, targets))


def test_eval_grid_dmma_form_in_subprocess(cuda):
    """The opt-in FP64 tensor-core form of the fused 13 -> 25 pair (CB_GRID_MODE=ws, read once per
    process) against the oracle: middle pair, padded last pair (q = 2) and a ragged last tile."""
    import os
    import subprocess
    import sys

    code = r"""
import numpy as np
import paper_2307_04688_b200 as cn
from oracle import cheb_oracle as orc
for shape, k in (((13, 13, 13, 13), (25, 25, 25, 25)), ((2, 13, 13), (3, 25, 25)), ((7, 3, 13, 13), (5, 4, 25, 25)),
                 ((13, 13, 3), (25, 25, 5))):
    rng = np.random.default_rng(sum(shape))
    coef = rng.standard_normal(shape)
    t = cn.CoefTensor([cn.make_basis(d - 1, -1.0, 1.0) for d in shape], coef)
    targets = [np.sort(rng.uniform(-1, 1, kk)) for kk in k]
    np.testing.assert_allclose(cn.eval_grid(t, targets), orc.eval_grid(coef, targets), rtol=1e-12, atol=1e-11)
print("ws ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CB_GRID_MODE="ws", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ws ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("shape,k", [((13, 13, 13, 13), (25, 25, 25, 25)), ((13, 13, 5, 5), (25, 25, 4, 4)),
                                     ((5, 4, 3, 6), (2, 3, 4, 5)), ((13,) * 6, (3, 2, 25, 25, 2, 3))])
def test_eval_grid_targets_vs_explicit_matrices(cuda, shape, k):
    """cb_eval_grid_targets (all evaluation matrices in one launch, one constant-bank upload for
    uniform 13 -> 25 grids) == cb_eval_grid on separately formed matrices (per-mode uploads),
    bitwise, and == the oracle."""
    import ctypes

    from paper_2307_04688_b200 import _lib
    from paper_2307_04688_b200.chebnd import _basis_device

    rng = np.random.default_rng(77 + len(shape))
    coef = rng.standard_normal(shape)
    t = cn.CoefTensor([cn.make_basis(d - 1, -1.0, 1.0) for d in shape], coef)
    targets = [np.linspace(-1, 1, kk) for kk in k]
    J = len(shape)
    lib = _lib.load()
    tdev = [_lib.to_device(x) for x in targets]
    Es = [_basis_device(tv, n, True) for tv, n in zip(tdev, shape)]  # separate allocations
    work_elems = int(lib.cb_eval_grid_workspace(J, _lib.i64_array(shape), _lib.i64_array(k)))
    work = _lib.empty((max(1, work_elems),))
    out_e = _lib.empty(tuple(k))
    eptrs = (ctypes.c_void_p * J)(*[_lib.ptr(e) for e in Es])
    _lib.check(lib.cb_eval_grid(J, _lib.i64_array(shape), _lib.ptr(t.device_coefficients), _lib.i64_array(k), eptrs,
                                _lib.ptr(out_e), _lib.ptr(work), work_elems, _lib.stream_handle()), "eval_grid")
    got_e = _lib.to_host(out_e)
    got = cn.eval_grid(t, targets)
    assert np.array_equal(got, got_e)
    close(got, orc.eval_grid(coef, targets))


def test_eval_grid_target_errors(cuda):
    t = cn.CoefTensor([cn.make_basis(4, -1.0, 1.0)] * 3, np.ones((5, 5, 5)))
    ok = np.linspace(-1, 1, 4)
    with pytest.raises(ValueError, match="outside"):
        cn.eval_grid(t, [ok, ok, np.array([0.0, 1.5])])
    with pytest.raises(ValueError, match="finite"):
        cn.eval_grid(t, [np.array([np.nan]), ok, ok])
    # within the clamp tolerance: clipped, no error
    close(cn.eval_grid(t, [ok, ok, np.array([1.0 + 5e-13])]), cn.eval_grid(t, [ok, ok, np.array([1.0])]))


@pytest.mark.parametrize("J,n,steps", [(2, 9, 7), (4, 5, 4), (6, 3, 3), (3, 17, 5), (4, 17, 2)])
def test_advect_loop(cuda, J, n, steps):
    rng = np.random.default_rng(1000 + J * n)
    A = rng.uniform(-0.5, 0.5, (J, J))
    axes = workloads.grid_axes(n, J)
    V0 = np.exp(sum(np.sin(np.pi * 1.3 * g) for g in np.meshgrid(*axes, indexing="ij")))
    got = cn.advect_loop(V0, bases_for(J, n), A, 0.01, steps)
    ref = orc.advect_loop(V0, A, 0.01, steps)
    close(got, ref)
    got_ng = cn.advect_loop(V0, bases_for(J, n), A, 0.01, steps, use_graph=False)
    assert np.array_equal(got, got_ng)


def test_advect_loop_counts_graph_replay_kernels(cuda):
    """cb_kernel_launches counts the kernels of every step-pair graph replay exactly like the
    eager launches of the same loop (bench.py's gpu_launches for the loop configs)."""
    from paper_2307_04688_b200 import _lib

    lib = _lib.load()
    J, n, steps = 3, 9, 8
    axes = workloads.grid_axes(n, J)
    V0 = np.exp(sum(np.sin(np.pi * g) for g in np.meshgrid(*axes, indexing="ij")))
    A = np.full((J, J), 0.1)
    cn.advect_loop(V0, bases_for(J, n), A, 0.01, steps)  # graph built here (captured launches not counted)
    c0 = lib.cb_kernel_launches()
    cn.advect_loop(V0, bases_for(J, n), A, 0.01, steps)
    c1 = lib.cb_kernel_launches()
    cn.advect_loop(V0, bases_for(J, n), A, 0.01, steps, use_graph=False)
    c2 = lib.cb_kernel_launches()
    assert c1 - c0 == c2 - c1 > 0


def test_advect_loop_config3_prefix(cuda):
    w = workloads.make("3", steps=3)
    got = cn.advect_loop(w.values, bases_for(w.J, w.n), w.A, w.dt, w.steps)
    close(got, orc.advect_loop(w.values, w.A, w.dt, w.steps))


def test_config5b_stepwise_oracle(cuda):
    """SURVEY §8(d) parity plan (i) for config 5b (J=6, n=13, full size): the GPU's V_t goes to the
    host, the oracle builds it (tensor_coeffs) and evaluates a seeded subset of 1,024 advected
    nodes; the GPU's V_{t+1} must match there, for t = 0 and t = 1."""
    w = workloads.make("5b")
    bases = bases_for(w.J, w.n)
    T, S = orc.advect_points(w.values.shape, w.A, w.dt)
    idx = np.sort(np.random.default_rng(55).choice(T.shape[0], 1024, replace=False))
    V = w.values
    for _ in range(2):
        V_next = cn.advect_loop(V, bases, w.A, w.dt, 1)
        ref = orc.eval_points(orc.tensor_coeffs(V), T[idx]) - S[idx]
        close(V_next.ravel()[idx], ref)
        V = V_next


def test_config5b_reduced_full_loop(cuda):
    """SURVEY §8(d) parity plan (ii): the full 20-step loop of config 5b at reduced n (J=6, n=5)."""
    w = workloads.make("5b", n=5)
    assert w.values.shape == (5,) * 6 and w.steps == 20
    got = cn.advect_loop(w.values, bases_for(w.J, w.n), w.A, w.dt, w.steps)
    close(got, orc.advect_loop(w.values, w.A, w.dt, w.steps))


def test_config4_full_batch_subset(cuda):
    """config 4 at its full M = 2^24 points on the GPU, checked against the oracle on a
    seeded subset of 2^14 point indices."""
    w = workloads.make("4")
    assert w.points.shape == (1 << 24, 5)
    t = cn.tensor_coeffs(w.values, bases_for(w.J, w.n))
    got = cn.eval_points(t, w.points)
    idx = np.sort(np.random.default_rng(44).choice(w.points.shape[0], 1 << 14, replace=False))
    ref = orc.eval_points_parallel(orc.tensor_coeffs(w.values), w.points[idx])
    close(got[idx], ref)


@pytest.mark.parametrize("cfg,M,n", [("1", 65_536, None), ("2", 4096, 9), ("4", 2048, 5)])
def test_build_eval_graph(cuda, cfg, M, n):
    """BuildEvalGraph (build + evaluate captured once, replayed) == the eager calls, bitwise, and
    follows in-place updates of its input buffers."""
    from paper_2307_04688_b200 import _lib
    from paper_2307_04688_b200.chebnd import _eval_points_device, tensor_coeffs_device

    w = workloads.make(cfg, M=M, n=n)
    shape = (w.n,) * w.J
    vals = _lib.to_device(w.values).clone()
    pts = _lib.to_device(w.points).clone()
    g = cn.BuildEvalGraph(shape, vals, pts)
    assert g.kernels_per_replay >= (1 if cfg == "1" else 2)   # config 1: one fused build + evaluate launch
    eager = _eval_points_device(shape, tensor_coeffs_device(vals, shape), pts, check=False)
    assert np.array_equal(_lib.to_host(g.replay()), _lib.to_host(eager))
    close(_lib.to_host(g.out), orc.eval_points(orc.tensor_coeffs(w.values), w.points))
    vals.mul_(2.0)
    pts.mul_(0.5)
    got = _lib.to_host(g.replay())
    close(got, orc.eval_points(orc.tensor_coeffs(2.0 * w.values), 0.5 * w.points))


@pytest.mark.parametrize("shape", [(33, 33, 33), (17,) * 4, (17,) * 5, (13,) * 6, (9,) * 5, (5,) * 7, (13,) * 3, (17, 17, 17)])
def test_group_build_bitwise_equals_per_mode_passes(cuda, shape):
    """The mode-group build (2 launches for equal modes n in {5, 9, 13, 17, 33}) applies the same
    per-fiber folded products in the same mode order (last mode first) as the one-pass-per-mode
    path, so the coefficients are bitwise identical; the per-mode path is reached here through
    two partial-axis transforms (cb_transform_axes over modes [k, J) then [0, k))."""
    from paper_2307_04688_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(len(shape) * 100 + shape[0])
    s = rng.standard_normal(shape)
    full = cn.tensor_coeffs(s, [cn.make_basis(d - 1, -1.0, 1.0) for d in shape]).coefficients
    J = len(shape)
    k = J // 2
    dev = _lib.to_device(s)
    mid = _lib.empty(shape)
    out = _lib.empty(shape)
    for (a0, a1, src, dst) in ((k, J, dev, mid), (0, k, mid, out)):
        _lib.check(lib.cb_transform_axes(J, _lib.i64_array(shape), a0, a1, _lib.ptr(src), _lib.ptr(dst), None, 0,
                                         _lib.stream_handle()), "transform_axes")
    per_mode = _lib.to_host(out)
    assert np.array_equal(full, per_mode), float(np.abs(full - per_mode).max())
    close(full, orc.tensor_coeffs(s))


# ------------------------------------------------------------------------------------------------
# the reference's input range: modes above 128 (large-mode transform), advected grids above 64
# nodes per mode (device node tables) — S/cheb1d.py:138-170 and S/chebnd.py:162-190 have no limits
# ------------------------------------------------------------------------------------------------

def test_transform_large_degrees_match_direct_sum(cuda):
    rng = np.random.default_rng(256)
    for N in (129, 150, 200, 255, 256, 511):
        s = rng.standard_normal(N + 1)
        c = cn.coeffs_from_samples(s, cn.make_basis(N, -1.0, 1.0)).coefficients
        np.testing.assert_allclose(c, orc.direct_transform(s), atol=1e-12)
        close(c, orc.cheb_transform(s))


@pytest.mark.parametrize("shape", [(200,), (130, 3), (3, 257), (150, 40), (40, 150, 2), (129, 34)])
def test_build_and_eval_large_modes(cuda, shape):
    rng = np.random.default_rng(sum(shape))
    s = rng.standard_normal(shape)
    bases = [cn.make_basis(d - 1, -1.0, 1.0) for d in shape]
    t = cn.tensor_coeffs(s, bases)
    C = orc.tensor_coeffs(s)
    close(t.coefficients, C)
    pts = 2.0 * rng.random((3000, len(shape))) - 1.0
    close(cn.eval_points(t, pts), orc.eval_points(C, pts))
    close(cn.eval_full(t, pts[0]), orc.eval_full(C, pts[0]))


def test_build_large_mode_rejects_nonfinite(cuda):
    s = np.ones((300,))
    s[17] = np.inf
    with pytest.raises(ValueError, match="finite"):
        cn.tensor_coeffs(s, [cn.make_basis(299, -1.0, 1.0)])


@pytest.mark.parametrize("shape,steps", [((100,), 4), ((70, 5), 3), ((5, 66, 3), 2)])
def test_advect_loop_above_64_nodes(cuda, shape, steps):
    J = len(shape)
    rng = np.random.default_rng(900 + sum(shape))
    A = rng.uniform(-0.5, 0.5, (J, J))
    axes = [workloads.grid_axes(n, 1)[0] for n in shape]
    V0 = np.exp(sum(np.sin(np.pi * 1.1 * g) for g in np.meshgrid(*axes, indexing="ij")))
    bases = [cn.make_basis(n - 1, 0.0, 1.0) for n in shape]
    got = cn.advect_loop(V0, bases, A, 0.01, steps)
    close(got, orc.advect_loop(V0, A, 0.01, steps))
    assert np.array_equal(got, cn.advect_loop(V0, bases, A, 0.01, steps, use_graph=False))


def test_build_nonfinite_with_null_status_does_not_fault(cuda):
    """cb_tensor_coeffs with a NaN sample and NO status block (the header allows NULL): the
    non-finite check is skipped instead of writing through a null pointer; the context stays
    usable (round-1 advice)."""
    import torch

    from paper_2307_04688_b200 import _lib

    lib = _lib.load()
    for shape in ((4, 4), (17,) * 4, (13,) * 3):
        s = np.ones(shape)
        s.flat[5] = np.nan
        dev = _lib.to_device(s)
        coef = _lib.empty((_lib.eval_layout(shape)["elems"],))
        _lib.check(lib.cb_tensor_coeffs(len(shape), _lib.i64_array(shape), _lib.ptr(dev), _lib.ptr(coef), None,
                                        _lib.stream_handle()), "tensor_coeffs")
        torch.cuda.synchronize()
    close(cn.tensor_coeffs(np.ones((3, 3)), bases_for(2, 3)).coefficients, orc.tensor_coeffs(np.ones((3, 3))))


def test_eval_advected_rejects_node_range_outside_grid(cuda):
    """cb_eval_advected(_peers) validate [node_begin, node_begin + count) against the grid before
    launching (the peers variant stores into other ranks' buffers)."""
    import ctypes

    from paper_2307_04688_b200 import _lib

    lib = _lib.load()
    shape = (5, 5)
    coef = _lib.empty((_lib.eval_layout(shape)["elems"],))
    out = _lib.empty((25,))
    A = _lib.dbl_array(np.zeros(4))
    lo, hi = _lib.dbl_array([0.0, 0.0]), _lib.dbl_array([1.0, 1.0])
    for begin, count in ((-1, 3), (20, 6), (0, 26), (3, -1)):
        rc = lib.cb_eval_advected(2, _lib.i64_array(shape), _lib.ptr(coef), begin, count, A, 0.01, lo, hi, 1,
                                  _lib.ptr(out), _lib.stream_handle())
        assert rc == 1 and b"node range" in lib.cb_last_error()
        dests = (ctypes.c_void_p * 1)(_lib.ptr(out))
        rc = lib.cb_eval_advected_peers(2, _lib.i64_array(shape), _lib.ptr(coef), begin, count, A, 0.01, lo, hi, 1,
                                        dests, 1, _lib.stream_handle())
        assert rc == 1 and b"node range" in lib.cb_last_error()
    assert lib.cb_eval_advected(2, _lib.i64_array(shape), _lib.ptr(coef), 20, 5, A, 0.01, lo, hi, 1, _lib.ptr(out),
                                _lib.stream_handle()) == 0


@pytest.mark.parametrize("shape", [(2,) * 9, (3,) * 10, (2, 3) * 6, (4, 3, 2, 2, 3, 2, 2, 3, 2)])
def test_more_than_eight_modes(cuda, shape):
    """J = 9..12 modes (the reference has no mode limit): build, scattered evaluation, eval_full,
    structured evaluation and the advected loop against the oracle."""
    J = len(shape)
    rng = np.random.default_rng(J * 31 + sum(shape))
    s = rng.standard_normal(shape)
    bases = [cn.make_basis(d - 1, -1.0, 1.0) for d in shape]
    t = cn.tensor_coeffs(s, bases)
    C = orc.tensor_coeffs(s)
    close(t.coefficients, C)
    pts = 2.0 * rng.random((777, J)) - 1.0
    close(cn.eval_points(t, pts), orc.eval_points(C, pts))
    close(cn.eval_full(t, pts[3]), orc.eval_full(C, pts[3]))
    targets = [np.linspace(-1, 1, 2 + (j % 2)) for j in range(J)]
    close(cn.eval_grid(t, targets), orc.eval_grid(C, targets))
    A = rng.uniform(-0.5, 0.5, (J, J))
    V0 = np.abs(s) + 1.0
    got = cn.advect_loop(V0, [cn.make_basis(d - 1, 0.0, 1.0) for d in shape], A, 0.01, 2)
    close(got, orc.advect_loop(V0, A, 0.01, 2))
