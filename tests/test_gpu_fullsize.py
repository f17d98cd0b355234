"""Full-size parity on the BASELINE configurations (SURVEY.md §8d parity plan): the CUDA path
against the pinned CPU oracle at the configs' real sizes and loop lengths, not reduced shapes.

* config 2: all 2^20 scattered points (S/solver.py:388-397 composition);
* config 3: the whole 100-step loop (S/solver.py:383-386, 441-449, 541-550), GPU and oracle run as
  two independent trajectories and compared at steps 1, 10, 25, 50, 75 and 100;
* config 5a: the full 13^6 -> 25^6 structured grid (J x eval_axis, S/chebnd.py:209-233), all
  244,140,625 values;
* config 5b: stepwise oracle at t = 0, 9 and 19 of the 20-step J=6 loop (GPU V_t -> oracle build
  + evaluation of 1,024 seeded advected nodes -> compared with the GPU's V_{t+1}).

Tolerance: allclose(rtol=1e-12, atol=1e-11) (BASELINE north star).  Every check prints its
max-abs and max-rel error (and the fraction of the tolerance used); with CB_PARITY_REPORT=<path>
the same records are appended there as JSON lines (profiles/parity_fullsize_r02.jsonl).
"""

import json
import os

import numpy as np
import pytest

import paper_2307_04688_b200 as cn
from oracle import cheb_oracle as orc
from paper_2307_04688_b200 import workloads

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-12, 1e-11
CORES = os.cpu_count() or 1


def _report(name, got, ref, **extra):
    """Chunked comparison (the 25^6 grid is 1.95 GB per side); returns the record."""
    got = np.asarray(got).ravel()
    ref = np.asarray(ref).ravel()
    assert got.shape == ref.shape
    max_abs = max_rel = used = 0.0
    bad = 0
    step = 1 << 24
    for s in range(0, got.size, step):
        g, r = got[s:s + step], ref[s:s + step]
        d = np.abs(g - r)
        ar = np.abs(r)
        max_abs = max(max_abs, float(d.max()))
        nz = ar > 0
        if nz.any():
            max_rel = max(max_rel, float((d[nz] / ar[nz]).max()))
        lim = ATOL + RTOL * ar
        used = max(used, float((d / lim).max()))
        bad += int(np.count_nonzero(d > lim))
    rec = {"check": name, "n": int(got.size), "max_abs": max_abs, "max_rel": max_rel,
           "tol_fraction_used": used, "violations": bad, "rtol": RTOL, "atol": ATOL, **extra}
    print(json.dumps(rec))
    path = os.environ.get("CB_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    assert bad == 0, rec
    return rec


def _bases(J, n):
    return [cn.make_basis(n - 1, 0.0, 1.0)] * J


def test_config2_all_points(cuda):
    w = workloads.make("2")
    assert w.points.shape == (1 << 20, 3)
    t = cn.tensor_coeffs(w.values, _bases(w.J, w.n))
    got = cn.eval_points(t, w.points)
    C = orc.tensor_coeffs(w.values)
    _report("config2_build", t.coefficients, C)
    ref = orc.eval_points_parallel(C, w.points, workers=CORES, block=4096)
    _report("config2_eval_all_2^20", got, ref)


def test_config3_full_100_steps(cuda):
    w = workloads.make("3")
    assert w.steps == 100 and w.values.shape == (17,) * 4
    bases = _bases(w.J, w.n)
    checkpoints = (1, 10, 25, 50, 75, 100)
    # GPU trajectory: segments of the device loop (state = V only, so segment restarts from the
    # host copy equal one uninterrupted loop bitwise; checked below on the first 10 steps)
    gpu = {}
    V = w.values
    t = 0
    for c in checkpoints:
        V = cn.advect_loop(V, bases, w.A, w.dt, c - t)
        t = c
        gpu[c] = V
    assert np.array_equal(cn.advect_loop(w.values, bases, w.A, w.dt, 10), gpu[10])
    # oracle trajectory, independent of the GPU's (errors accumulate separately on each side)
    pts = orc.advect_points(w.values.shape, w.A, w.dt)
    R = w.values
    for s in range(1, w.steps + 1):
        R = orc.advect_step(R, w.A, w.dt, points=pts, workers=CORES, block=2048)
        if s in gpu:
            _report(f"config3_step{s}", gpu[s], R, step=s)


def test_config5a_full_grid(cuda):
    w = workloads.make("5a")
    assert w.values.shape == (13,) * 6 and len(w.targets) == 6 and w.targets[0].size == 25
    t = cn.tensor_coeffs(w.values, _bases(w.J, w.n))
    got = cn.eval_grid(t, w.targets)
    assert got.shape == (25,) * 6
    C = orc.tensor_coeffs(w.values)
    _report("config5a_build", t.coefficients, C)
    ref = orc.eval_grid(C, w.targets)
    _report("config5a_grid_25^6", got, ref)


def test_config5b_stepwise_t0_t9_t19(cuda):
    w = workloads.make("5b")
    assert w.steps == 20
    bases = _bases(w.J, w.n)
    T, S = orc.advect_points(w.values.shape, w.A, w.dt)
    idx = np.sort(np.random.default_rng(55).choice(T.shape[0], 1024, replace=False))
    V = w.values
    t = 0
    for target in (0, 9, 19):
        if target > t:
            V = cn.advect_loop(V, bases, w.A, w.dt, target - t)
            t = target
        V_next = cn.advect_loop(V, bases, w.A, w.dt, 1)
        ref = orc.eval_points_parallel(orc.tensor_coeffs(V), T[idx], workers=CORES, block=64) - S[idx]
        _report(f"config5b_step{target}->{target + 1}", V_next.ravel()[idx], ref, step=target)
        V = V_next
        t += 1


def test_config5a_grid_nonsymmetric_targets(cuda):
    """The J = 6 13 -> 25 plan on targets that are NOT symmetric about 0 (the unfolded kernels),
    full 25^6 grid against the oracle."""
    w = workloads.make("5a")
    rng = np.random.default_rng(5150)
    targets = [np.sort(2.0 * rng.random(25) - 1.0) for _ in range(6)]
    t = cn.tensor_coeffs(w.values, _bases(w.J, w.n))
    got = cn.eval_grid(t, targets)
    ref = orc.eval_grid(orc.tensor_coeffs(w.values), targets)
    _report("config5a_grid_25^6_nonsymmetric_targets", got, ref)
