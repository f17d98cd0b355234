"""CPU oracle for the tensor-Chebyshev hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.  The product
package ``paper_2307_04688_b200`` never imports it and has no CPU fallback.

It restates, in numpy, the algorithm of the reference package ``chebnash`` 0.1.0
(``/root/reference/pkg/src/chebnash``, cited as ``S/<file>:<line>``), which itself runs on numpy's
pocketfft (``np.fft.rfft``) and OpenBLAS (``np.matmul``).  Each function names the reference
lines it follows.  Parity of this restatement with the reference is PINNED by
``tests/test_oracle_golden.py`` against fixtures in ``tests/golden/`` that
``tests/golden/make_golden.py`` produced by importing the reference itself, and against the
reference's own known-answer tests (direct cosine sum, constants, T1 x T1, separable products).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CLAMP_TOL = 1e-12  # S/cheb1d.py:22


# ---------------------------------------------------------------------------------------------
# 1-D machinery
# ---------------------------------------------------------------------------------------------

def reference_nodes(degree: int) -> np.ndarray:
    """cos(pi k / N), k = 0..N, descending, ends pinned (S/cheb1d.py:107-114)."""
    if degree == 0:
        return np.zeros(1)
    out = np.cos(np.pi * np.arange(degree + 1) / degree)
    out[0], out[-1] = 1.0, -1.0
    return out


def interval_nodes(degree: int, a: float, b: float) -> np.ndarray:
    """make_basis nodes on [a, b] (S/cheb1d.py:97-103)."""
    if degree == 0:
        return np.array([0.5 * (a + b)])
    k = np.arange(degree + 1)
    x = 0.5 * (b - a) * np.cos(np.pi * k / degree) + 0.5 * (a + b)
    x[0], x[-1] = b, a
    return x


def clamp_reference(x, tol: float = CLAMP_TOL) -> np.ndarray:
    """Clip to [-1, 1]; non-finite or beyond tol raises ValueError (S/cheb1d.py:127-135)."""
    x = np.asarray(x, dtype=float)
    if not np.isfinite(x).all():
        raise ValueError("evaluation points must be finite")
    ax = np.abs(x)
    if (ax > 1.0 + tol).any():
        raise ValueError(f"evaluation point outside [-1, 1] beyond tolerance: |x| = {float(ax.max())}")
    return np.clip(x, -1.0, 1.0)


def cheb_transform(values, axis: int = 0) -> np.ndarray:
    """DCT-I via the real FFT of the even extension, ends halved (S/cheb1d.py:138-170)."""
    v = np.moveaxis(np.asarray(values, dtype=float), axis, 0)
    N = v.shape[0] - 1
    if N < 0:
        raise ValueError("need at least one sample")
    if N == 0:
        return np.moveaxis(v.copy(), 0, axis)
    mirrored = np.concatenate((v, v[N - 1:0:-1]), axis=0)          # length 2N
    c = np.fft.rfft(mirrored, axis=0).real / N                       # N + 1 rows
    c[0] *= 0.5
    c[N] *= 0.5
    return np.moveaxis(c, 0, axis)


def direct_transform(samples) -> np.ndarray:
    """O(N^2) cosine sum with halved end samples — the reference tests' own oracle
    (T/test_cheb1d.py:18-29, T/test_acceptance.py:81-96)."""
    s = np.asarray(samples, dtype=float)
    N = s.size - 1
    if N == 0:
        return s.copy()
    k = np.arange(N + 1)
    w = np.ones(N + 1)
    w[[0, N]] = 0.5
    scale = np.full(N + 1, 2.0 / N)
    scale[[0, N]] = 1.0 / N
    return scale * (np.cos(np.pi * np.outer(k, k) / N) @ (w * s))


def transform_matrix(degree: int) -> np.ndarray:
    """M0 = diag(s) B(ref nodes)^T diag(w) (S/solver.py:162-171)."""
    size = degree + 1
    B = row_basis(reference_nodes(degree), size)
    w = np.ones(size)
    w[[0, -1]] = 0.5
    s = np.full(size, 2.0 / degree)
    s[[0, -1]] = 1.0 / degree
    return s[:, None] * B.T * w[None, :]


def row_basis(x, size: int) -> np.ndarray:
    """B[p, l] = T_l(x_p) by the three-term recurrence (S/chebnd.py:135-144)."""
    x = np.asarray(x, dtype=float).ravel()
    B = np.empty((x.size, size))
    B[:, 0] = 1.0
    if size > 1:
        B[:, 1] = x
    for l in range(2, size):
        B[:, l] = 2.0 * x * B[:, l - 1] - B[:, l - 2]
    return B


def clenshaw(c, x) -> np.ndarray:
    """Backward Clenshaw over the leading axis (S/cheb1d.py:198-214)."""
    c = np.asarray(c, dtype=float)
    x = np.asarray(x, dtype=float)
    N = c.shape[0] - 1
    if N == 0:
        return np.broadcast_to(c[0], np.broadcast_shapes(c[0].shape, x.shape)).copy()
    b1 = np.zeros(np.broadcast_shapes(c.shape[1:], x.shape))
    b2 = np.zeros_like(b1)
    for k in range(N, 0, -1):
        b1, b2 = c[k] + 2.0 * x * b1 - b2, b1
    return c[0] + x * b1 - b2


def derivative_array(p) -> np.ndarray:
    """Coefficient-space derivative along the last axis (S/cheb1d.py:230-249)."""
    p = np.asarray(p, dtype=float)
    n = p.shape[-1] - 1
    q = np.zeros(p.shape[:-1] + (n,))
    q[..., n - 1] = 2.0 * n * p[..., n]
    if n >= 2:
        q[..., n - 2] = 2.0 * (n - 1) * p[..., n - 1]
    for l in range(n - 3, -1, -1):
        q[..., l] = q[..., l + 2] + 2.0 * (l + 1) * p[..., l + 1]
    q[..., 0] *= 0.5
    return q


# ---------------------------------------------------------------------------------------------
# tensor build and evaluation
# ---------------------------------------------------------------------------------------------

def tensor_coeffs(samples) -> np.ndarray:
    """Algorithm Cnv: transform axis 0, rotate, J times (S/chebnd.py:162-190)."""
    s = np.asarray(samples, dtype=float)
    if not np.isfinite(s).all():
        raise ValueError("samples must be finite")
    J = s.ndim
    for _ in range(J):
        s = np.moveaxis(cheb_transform(s, 0), 0, J - 1)
    return np.ascontiguousarray(s)


def stack_coeffs(samples) -> np.ndarray:
    """Same transform on the leading J axes of a (n..., N_P) stack (S/chebnd.py:193-206)."""
    s = np.asarray(samples, dtype=float)
    J = s.ndim - 1
    for _ in range(J):
        s = np.moveaxis(cheb_transform(s, 0), 0, J - 1)
    return np.ascontiguousarray(s)


def eval_points(coef, pts, block: int = 4096) -> np.ndarray:
    """Scattered evaluation, the solver composition S/solver.py:388-397:
    first-mode row-by-row contraction (_bind_rows S/chebnd.py:152-154), per-point diagonal
    contractions of the middle modes (_bind_diagonal :157-159), last-mode einsum.  `pts` are
    pre-clamped reference coordinates (M, J); processed in blocks of `block` points like the
    solver's node blocks (S/solver.py:61-87)."""
    coef = np.asarray(coef, dtype=float)
    pts = np.asarray(pts, dtype=float)
    J = coef.ndim
    sizes = coef.shape
    M = pts.shape[0]
    out = np.empty(M)
    if J == 1:
        for s in range(0, M, block):
            B = row_basis(pts[s:s + block, 0], sizes[0])
            out[s:s + block] = np.einsum("ql,l->q", B, coef)
        return out
    flat = coef.reshape(sizes[0], -1)
    for s in range(0, M, block):
        p = pts[s:s + block]
        m = p.shape[0]
        B = row_basis(p[:, 0], sizes[0])
        cur = np.matmul(B[:, None, :], flat)[:, 0, :]                       # (m, n^{J-1})
        for d in range(1, J - 1):
            B = row_basis(p[:, d], sizes[d])
            cur = np.matmul(B[:, None, :], cur.reshape(m, sizes[d], -1))[:, 0, :]
        B = row_basis(p[:, J - 1], sizes[J - 1])
        out[s:s + m] = np.einsum("ql,ql->q", B, cur.reshape(m, sizes[J - 1]))
    return out


def eval_points_parallel(coef, pts, workers: int | None = None, block: int = 1024) -> np.ndarray:
    """The reference's block-parallel scheme (S/solver.py:423-437): disjoint point blocks on a
    ThreadPoolExecutor; numpy releases the GIL inside matmul."""
    pts = np.asarray(pts, dtype=float)
    M = pts.shape[0]
    workers = workers or os.cpu_count() or 1
    out = np.empty(M)
    chunks = [(s, min(M, s + block)) for s in range(0, M, block)]

    def run(ch):
        a, b = ch
        out[a:b] = eval_points(coef, pts[a:b], block=block)

    if workers <= 1:
        for ch in chunks:
            run(ch)
    else:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(run, chunks))
    return out


def eval_full(coef, point) -> float:
    """Nested Clenshaw over all axes at one point (S/chebnd.py:315-327)."""
    x = clamp_reference(point)
    c = np.asarray(coef, dtype=float)
    for xi in x:
        c = clenshaw(c, xi)
    return float(c)


def eval_axis(coef, points) -> np.ndarray:
    """Bind the leading axis at shared points, rotate (S/chebnd.py:209-233): (rest..., k)."""
    x = clamp_reference(points)
    c = np.asarray(coef, dtype=float)
    B = row_basis(x, c.shape[0])
    out = np.matmul(B[:, None, :], c.reshape(c.shape[0], -1))[:, 0, :]
    return np.moveaxis(out.reshape((x.size,) + c.shape[1:]), 0, -1)


def eval_axis_stack(coef, points) -> np.ndarray:
    """Stack form (S/chebnd.py:234-240): (rest..., k, N_P)."""
    x = clamp_reference(points)
    A = np.asarray(coef, dtype=float)
    d1, m = A.shape[0], A.shape[-1]
    rest = A.shape[1:-1]
    Am = np.ascontiguousarray(np.moveaxis(A, -1, 0)).reshape(m, d1, -1)
    B = row_basis(x, d1)
    out = np.matmul(B, Am)                                           # (m, k, rest)
    out = np.moveaxis(out, 0, -1).reshape((x.size,) + rest + (m,))
    return np.moveaxis(out, 0, -2)


def eval_diagonal(coef, points) -> np.ndarray:
    """Member j bound at its own point x_j (S/chebnd.py:275-312): (rest..., N_P)."""
    x = clamp_reference(points)
    A = np.asarray(coef, dtype=float)
    d1, m = A.shape[0], A.shape[-1]
    rest = A.shape[1:-1]
    Am = np.ascontiguousarray(np.moveaxis(A, -1, 0)).reshape(m, d1, -1)
    B = row_basis(x, d1)
    out = np.matmul(B[:, None, :], Am)[:, 0, :]
    return np.moveaxis(out.reshape((m,) + rest), 0, -1)


def gather_index(member_shape, count: int) -> np.ndarray:
    """Flat dimension-1-fastest selection of the diagonal (S/chebnd.py:243-272)."""
    rest = int(np.prod(member_shape[1:], dtype=np.int64)) if len(member_shape) > 1 else 1
    r = np.arange(rest, dtype=np.int64)
    m = np.arange(count, dtype=np.int64)
    return (r[:, None] + rest * (count + 1) * m[None, :]).ravel(order="F")


def eval_grid(coef, targets) -> np.ndarray:
    """Structured evaluation: J successive eval_axis products; targets[j] are
    reference coordinates along dim j.  Output (k_1, ..., k_J)."""
    cur = np.asarray(coef, dtype=float)
    for t in targets:
        cur = eval_axis(cur, t)
    return cur


# ---------------------------------------------------------------------------------------------
# time loop (BASELINE configs 3 / 5b): the solver skeleton S/solver.py:383-386, 441-449, 541-550
# with a fixed linear drift
# ---------------------------------------------------------------------------------------------

def grid_nodes(n_per_dim, lo=0.0, hi=1.0) -> list[np.ndarray]:
    return [interval_nodes(n - 1, lo, hi) for n in n_per_dim]


def advect_points(n_per_dim, A, dt, lo=0.0, hi=1.0):
    """Advected grid nodes in reference coordinates and the source term, C-order node
    enumeration: y = clip(x + dt A x, lo, hi), t = (2y - (lo+hi)) / (hi - lo), s = dt |x|^2."""
    axes = grid_nodes(n_per_dim, lo, hi)
    X = np.stack([g.ravel() for g in np.meshgrid(*axes, indexing="ij")], axis=-1)
    Y = np.clip(X + dt * (X @ np.asarray(A, dtype=float).T), lo, hi)
    T = np.clip((2.0 * Y - (lo + hi)) / (hi - lo), -1.0, 1.0)
    S = dt * np.sum(X * X, axis=1)
    return T, S


def advect_step(values, A, dt, lo=0.0, hi=1.0, points=None, block: int = 4096, workers: int = 1):
    """One step V <- eval(tensor_coeffs(V), advected nodes) - dt |x|^2."""
    V = np.asarray(values, dtype=float)
    if points is None:
        points = advect_points(V.shape, A, dt, lo, hi)
    T, S = points
    C = tensor_coeffs(V)
    if workers > 1:
        v = eval_points_parallel(C, T, workers=workers, block=block)
    else:
        v = eval_points(C, T, block=block)
    return (v - S).reshape(V.shape)


def advect_loop(values, A, dt, steps: int, lo=0.0, hi=1.0, workers: int = 1):
    V = np.asarray(values, dtype=float)
    pts = advect_points(V.shape, A, dt, lo, hi)
    for _ in range(steps):
        V = advect_step(V, A, dt, lo, hi, points=pts, workers=workers)
    return V
