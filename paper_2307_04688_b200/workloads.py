"""Seeded synthetic inputs for the five BASELINE.json configurations (host-side input synthesis).

No public dataset is involved: every BASELINE input is synthetic.  Conventions:
grid = make_basis(n-1, 0, 1) per dim (descending Chebyshev-Lobatto nodes, S/cheb1d.py:73-104),
node values sampled at np.meshgrid(..., indexing="ij") in C order, points uniform in [0, 1]^J
mapped to reference coordinates t = 2x - 1, RNG = np.random.default_rng(20240801 + cfg) with the
draw order: function parameters -> drift matrix -> points (one (M, J) call).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_BASE = 20240801


def grid_axes(n: int, J: int, lo: float = 0.0, hi: float = 1.0) -> list[np.ndarray]:
    N = n - 1
    k = np.arange(n)
    x = 0.5 * (hi - lo) * np.cos(np.pi * k / N) + 0.5 * (lo + hi)
    x[0], x[-1] = hi, lo
    return [x.copy() for _ in range(J)]


def _sin_family(axes, a):
    grids = np.meshgrid(*axes, indexing="ij")
    return np.exp(sum(np.sin(np.pi * a[j] * grids[j]) for j in range(len(axes))))


def _gauss_family(axes, b, c):
    grids = np.meshgrid(*axes, indexing="ij")
    return np.exp(-sum(b[j] * (grids[j] - c[j]) ** 2 for j in range(len(axes))))


@dataclass
class Workload:
    cfg: str
    J: int
    n: int
    values: np.ndarray            # (n,)*J node values (C order)
    points: np.ndarray | None     # (M, J) reference coordinates, scattered configs
    A: np.ndarray | None          # drift matrix, loop configs
    dt: float
    steps: int
    targets: list | None          # per-dim reference target coordinates, structured config
    params: dict

    @property
    def M(self) -> int:
        if self.points is not None:
            return int(self.points.shape[0])
        return int(self.n ** self.J)


def make(cfg: str, M: int | None = None, n: int | None = None, steps: int | None = None) -> Workload:
    """Build config `cfg` in {"1","2","3","4","5a","5b"}.  M / n / steps override the BASELINE
    sizes (used for reduced parity cases); the RNG stream is unchanged."""
    cfg = str(cfg)
    key = {"1": 1, "2": 2, "3": 3, "4": 4, "5a": 5, "5b": 5}[cfg]
    rng = np.random.default_rng(SEED_BASE + key)
    if cfg == "1":
        J, nn = 2, n or 17
        a = rng.uniform(0.5, 2.0, J)
        axes = grid_axes(nn, J)
        vals = _sin_family(axes, a)
        M = M or 65_536
        pts = 2.0 * rng.random((M, J)) - 1.0
        return Workload(cfg, J, nn, vals, pts, None, 0.0, 0, None, {"a": a})
    if cfg == "2":
        J, nn = 3, n or 33
        b = rng.uniform(1.0, 5.0, J)
        c = rng.uniform(0.0, 1.0, J)
        axes = grid_axes(nn, J)
        vals = _gauss_family(axes, b, c)
        M = M or (1 << 20)
        pts = 2.0 * rng.random((M, J)) - 1.0
        return Workload(cfg, J, nn, vals, pts, None, 0.0, 0, None, {"b": b, "c": c})
    if cfg == "3":
        J, nn = 4, n or 17
        a = rng.uniform(0.5, 2.0, J)
        A = rng.uniform(-0.5, 0.5, (J, J))
        axes = grid_axes(nn, J)
        vals = _sin_family(axes, a)
        return Workload(cfg, J, nn, vals, None, A, 0.01, steps or 100, None, {"a": a})
    if cfg == "4":
        J, nn = 5, n or 17
        a = rng.uniform(0.5, 2.0, J)
        axes = grid_axes(nn, J)
        vals = _sin_family(axes, a)
        M = M or (1 << 24)
        pts = 2.0 * rng.random((M, J)) - 1.0
        return Workload(cfg, J, nn, vals, pts, None, 0.0, 0, None, {"a": a})
    # config 5: J=6, n=13, gaussian family; 5a structured grid, 5b 20-step loop
    J, nn = 6, n or 13
    b = rng.uniform(1.0, 5.0, J)
    c = rng.uniform(0.0, 1.0, J)
    A = rng.uniform(-0.5, 0.5, (J, J))
    axes = grid_axes(nn, J)
    vals = _gauss_family(axes, b, c)
    if cfg == "5a":
        k = M or 25  # targets per dim (builder's choice, recorded in DESIGN.md)
        t = 2.0 * np.linspace(0.0, 1.0, k) - 1.0
        return Workload(cfg, J, nn, vals, None, None, 0.0, 0, [t.copy() for _ in range(J)], {"b": b, "c": c, "k": k})
    return Workload(cfg, J, nn, vals, None, A, 0.01, steps or 20, None, {"b": b, "c": c})
