"""Generate the golden fixtures in tests/golden/ by running the REFERENCE implementation itself.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference package (chebnash 0.1.0, pure Python + numpy) is imported read-only from
/root/reference/pkg/src; every output stored here is produced by its own public functions or by
the solver's private evaluation kernels composed exactly as S/solver.py:388-397 composes them.
Inputs are seeded; the fixtures pin both the CPU oracle (tests/test_oracle_golden.py) and the CUDA
path (tests/test_gpu_golden.py).  /root/reference does not exist on the GPU box, so the fixtures
(not the reference) travel with the repo.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("CHEBNASH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import chebnash as ref  # noqa: E402
from chebnash.chebnd import _bind_diagonal, _bind_rows, _row_basis  # noqa: E402

from paper_2307_04688_b200 import workloads  # noqa: E402  (seeded input synthesis only)


def solver_eval(coef: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """The reference's batched value evaluation, S/solver.py:390-397, on pre-clamped points."""
    J = coef.ndim
    sizes = coef.shape
    B = _row_basis(pts[:, 0], sizes[0])
    if J == 1:
        return np.einsum("ql,l->q", B, coef)
    curv = _bind_rows(B, coef.reshape(sizes[0], -1))
    for d in range(1, J - 1):
        B = _row_basis(pts[:, d], sizes[d])
        curv = _bind_diagonal(B, curv.reshape(-1, sizes[d], curv.shape[1] // sizes[d]))
    B = _row_basis(pts[:, J - 1], sizes[J - 1])
    return np.einsum("ql,ql->q", B, curv.reshape(-1, sizes[J - 1]))


def ref_advect(values: np.ndarray, A: np.ndarray, dt: float, steps: int) -> np.ndarray:
    """Loop skeleton of S/solver.py:383-386 + 441-449 with a fixed linear drift, reference calls only."""
    J = values.ndim
    bases = [ref.make_basis(n - 1, 0.0, 1.0) for n in values.shape]
    grids = np.meshgrid(*(b.nodes for b in bases), indexing="ij")
    X = np.stack([g.ravel() for g in grids], axis=-1)
    Y = np.clip(X + dt * (X @ A.T), 0.0, 1.0)
    T = np.stack([ref.to_reference(bases[d], Y[:, d]) for d in range(J)], axis=-1)
    T = np.clip(T, -1.0, 1.0)
    S = dt * np.sum(X * X, axis=1)
    V = values
    for _ in range(steps):
        C = ref.tensor_coeffs(V, bases).coefficients
        V = (solver_eval(C, T) - S).reshape(values.shape)
    return V


def main():
    out = {}
    rng = np.random.default_rng(20240801)

    # 1-D transforms, N = 0..64 (T/test_cheb1d.py:253-259 range)
    for n in range(0, 65):
        s = rng.standard_normal(n + 1)
        out[f"t1d_in_{n}"] = s
        out[f"t1d_out_{n}"] = ref.coeffs_from_samples(s, ref.make_basis(n, -1.0, 1.0)).coefficients
    blk = rng.standard_normal((9, 5, 4))
    out["taxis_in"] = blk
    for ax in range(3):
        out[f"taxis_out_{ax}"] = ref.cheb1d.cheb_transform(blk, axis=ax)

    # tensor builds + scattered evaluation at BASELINE-family shapes (reduced where the reference is slow)
    cases = {
        "c1": workloads.make("1", M=256),
        "c2": workloads.make("2", M=256, n=9),
        "c3": workloads.make("3", n=5),
        "c4": workloads.make("4", M=256, n=5),
        "c5": workloads.make("5a", n=3),
    }
    for key, w in cases.items():
        vals = w.values
        bases = [ref.make_basis(n - 1, 0.0, 1.0) for n in vals.shape]
        C = ref.tensor_coeffs(vals, bases).coefficients
        out[f"{key}_values"] = vals
        out[f"{key}_coef"] = C
        pts = w.points if w.points is not None else 2.0 * np.random.default_rng(5).random((256, vals.ndim)) - 1.0
        pts = np.clip(pts, -1.0, 1.0)
        out[f"{key}_points"] = pts
        out[f"{key}_eval"] = solver_eval(C, pts)
        out[f"{key}_evalfull"] = np.array([ref.eval_full(ref.tensor_coeffs(vals, bases), p) for p in pts[:8]])

    # ragged shapes on [-1, 1]
    for i, shape in enumerate([(4, 5, 6), (3, 2), (2, 3, 2, 3), (7,), (1, 4, 1), (6, 6, 6, 6, 2)]):
        s = rng.standard_normal(shape)
        bases = [ref.make_basis(n - 1, -1.0, 1.0) for n in shape]
        C = ref.tensor_coeffs(s, bases).coefficients
        pts = rng.uniform(-1.0, 1.0, (64, len(shape)))
        out[f"r{i}_values"] = s
        out[f"r{i}_coef"] = C
        out[f"r{i}_points"] = pts
        out[f"r{i}_eval"] = solver_eval(C, pts)

    # axis / stack / diagonal / gather API
    sc = rng.standard_normal((5, 3, 4, 6))
    sbases = [ref.make_basis(n - 1, -1.0, 1.0) for n in sc.shape[:-1]]
    st = ref.TensorStack(sbases, sc)
    spts = rng.uniform(-1.0, 1.0, 6)
    g = ref.make_gather_index(sc.shape[:-1], 6)
    out["stack_coef"] = sc
    out["stack_points"] = spts
    out["stack_axis"] = ref.eval_axis(st, spts)
    out["stack_diag"] = ref.eval_diagonal_batch(st, spts, g).coefficients
    out["stack_gather_flat"] = g.flat
    out["stack_gather_take"] = g.take(ref.eval_axis(st, spts))
    ssamp = rng.standard_normal((4, 5, 3))
    out["stackc_in"] = ssamp
    out["stackc_out"] = ref.stack_coeffs(ssamp, [ref.make_basis(3, -1, 1), ref.make_basis(4, -1, 1)]).coefficients
    tc = rng.standard_normal((5, 4, 3))
    tt = ref.CoefTensor([ref.make_basis(n - 1, -1.0, 1.0) for n in tc.shape], tc)
    tpts = rng.uniform(-1.0, 1.0, 7)
    out["axis_coef"] = tc
    out["axis_points"] = tpts
    out["axis_out"] = ref.eval_axis(tt, tpts)
    bpts = np.linspace(-1.0, 1.0, 9)
    out["basis_points"] = bpts
    out["basis_out"] = ref.basis_matrix(bpts, 6)
    # structured grid: J successive eval_axis products
    targets = [np.linspace(-1.0, 1.0, k) for k in (4, 3, 5)]
    cur = tt.coefficients
    for t in targets:
        cur = ref.eval_axis(ref.CoefTensor([ref.make_basis(n - 1, -1.0, 1.0) for n in cur.shape], cur), t)
    out["grid_out"] = cur
    for j, t in enumerate(targets):
        out[f"grid_t{j}"] = t

    # time loop (BASELINE configs 3 / 5b family) with reference calls only
    for key, (J, n, steps) in {"loopa": (2, 9, 5), "loopb": (3, 5, 3), "loopc": (4, 5, 2)}.items():
        r2 = np.random.default_rng(1000 + J * n)
        A = r2.uniform(-0.5, 0.5, (J, J))
        axes = workloads.grid_axes(n, J)
        V0 = np.exp(sum(np.sin(np.pi * 1.3 * gg) for gg in np.meshgrid(*axes, indexing="ij")))
        out[f"{key}_V0"] = V0
        out[f"{key}_A"] = A
        out[f"{key}_steps"] = np.array(steps)
        out[f"{key}_V"] = ref_advect(V0, A, 0.01, steps)
    # config 3 at full size for 2 steps: store seeded sample entries + the full sum
    w3 = workloads.make("3", steps=2)
    V3 = ref_advect(w3.values, w3.A, w3.dt, 2)
    idx = np.random.default_rng(3).choice(V3.size, 4096, replace=False)
    out["c3full_idx"] = idx
    out["c3full_V2_sample"] = V3.ravel()[idx]
    out["c3full_V2_sum"] = np.array(V3.sum())

    np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
