"""CPU: the C-ABI library loads without a GPU, exports every symbol include/chebnash_b200.h declares,
and its host-side planning / validation behaves; the Python shim refuses to compute without CUDA
(no CPU fallback).  No kernel is launched here."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2307_04688_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chebnash_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes signature table covers exactly the header
    assert sorted(_lib.SIGNATURES) == syms


def test_abi_version_and_cpu_runtime_info():
    lib = _lib.load()
    assert lib.cb_abi_version() == 1
    vals = [ctypes.c_int(-1) for _ in range(4)]
    assert lib.cb_runtime_info(*[ctypes.byref(v) for v in vals]) == 0
    assert vals[0].value >= 0  # 0 devices on the CPU container


@pytest.mark.parametrize("shape,q,K,Kp,R,R8", [
    ((17, 17), 1, 17, 20, 17, 24),
    ((33, 33, 33), 1, 33, 36, 1089, 1096),
    ((17,) * 4, 2, 289, 292, 289, 296),
    ((17,) * 5, 2, 289, 292, 4913, 4920),
    ((13,) * 6, 2, 169, 172, 28561, 28568),
])
def test_eval_layout_plan(shape, q, K, Kp, R, R8):
    L = _lib.eval_layout(shape)
    assert (L["q"], L["K"], L["Kp"], L["R"], L["R8"]) == (q, K, Kp, R, R8)
    assert L["elems"] == R8 * Kp


def test_eval_layout_properties_random():
    rng = np.random.default_rng(0)
    for _ in range(200):
        J = int(rng.integers(1, 7))
        shape = tuple(int(x) for x in rng.integers(1, 20, J))
        L = _lib.eval_layout(shape)
        assert L["K"] * L["R"] == int(np.prod(shape))
        assert L["Kp"] % 4 == 0 and L["Kp"] >= L["K"] and L["Kp"] - L["K"] < 4
        assert L["R8"] % 8 == 0 and L["R8"] >= L["R"] and L["R8"] - L["R"] < 8
        assert 1 <= L["q"] <= J


def test_invalid_arguments_map_to_valueerror():
    lib = _lib.load()
    out = (ctypes.c_int64 * 6)()
    rc = lib.cb_eval_layout(0, _lib.i64_array([1]), out)
    assert rc == 1 and b"modes" in lib.cb_last_error()
    rc = lib.cb_eval_layout(2, _lib.i64_array([3, 0]), out)
    assert rc == 1
    with pytest.raises(ValueError):
        _lib.check(rc)
    rc = lib.cb_eval_layout(1, _lib.i64_array([5000]), out)
    assert rc == 1 and b"4096" in lib.cb_last_error()
    # degree 255 (mode size 256) is in range since the large-mode transform path
    assert lib.cb_eval_layout(1, _lib.i64_array([256]), out) == 0


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2307_04688_b200 as cn

    b = cn.make_basis(4, 0.0, 1.0)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cn.tensor_coeffs(np.ones((5, 5)), [b, b])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cn.coeffs_from_samples(np.ones(5), b)


def test_host_metadata_matches_reference_conventions():
    import paper_2307_04688_b200 as cn

    b = cn.make_basis(4, -1.0, 1.0)
    r = np.sqrt(2.0) / 2.0
    np.testing.assert_allclose(b.nodes, [1.0, r, 0.0, -r, -1.0], atol=1e-15)
    assert not b.nodes.flags.writeable
    b9 = cn.make_basis(9, 0.3, 4.7)
    assert b9.nodes[0] == 4.7 and b9.nodes[-1] == 0.3 and np.all(np.diff(b9.nodes) < 0)
    np.testing.assert_allclose(cn.make_basis(0, 2.0, 4.0).nodes, [3.0])
    for a, bb in [(1.0, 1.0), (2.0, -1.0), (np.nan, 1.0), (0.0, np.inf)]:
        with pytest.raises(ValueError):
            cn.make_basis(3, a, bb)
    with pytest.raises(ValueError):
        cn.make_basis(-1, 0.0, 1.0)
    x = np.linspace(-2.0, 7.0, 13)
    b5 = cn.make_basis(5, -2.0, 7.0)
    np.testing.assert_allclose(cn.from_reference(b5, cn.to_reference(b5, x)), x, atol=1e-14)
    with pytest.raises(ValueError):
        cn.clamp_reference([1.0 + 1e-9])
    assert cn.clamp_reference(1.0 + 1e-13) == 1.0


def test_workloads_are_seeded_and_shaped():
    from paper_2307_04688_b200 import workloads

    a = workloads.make("2", M=100)
    b = workloads.make("2", M=100)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.points, b.points)
    assert a.values.shape == (33, 33, 33) and a.points.shape == (100, 3)
    assert np.all(np.abs(a.points) <= 1.0)
    w3 = workloads.make("3")
    assert w3.values.shape == (17,) * 4 and w3.A.shape == (4, 4) and w3.steps == 100 and w3.dt == 0.01
    w5 = workloads.make("5a")
    assert len(w5.targets) == 6 and w5.targets[0].size == 25
