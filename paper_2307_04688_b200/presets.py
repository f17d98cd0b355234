"""Named experiment configurations of the reference (S/presets.py): the paper's three spatial
layouts with the shared parameter set beta = phi = 1, A = c = 0.5 (zero-row-sum exchange)."""

from __future__ import annotations

import numpy as np

from .game import GameSpec

PRESET_NAMES = ("example1", "example3", "example4")

_LAYOUTS = {
    # two players, one common boundary
    "example1": dict(J=2, K=[[-1.0, 1.0], [1.0, -1.0]], Np=8, Nu=8),
    # three players in a chain
    "example3": dict(J=3, K=[[-1.0, 1.0, 0.0], [1.0, -2.0, 1.0], [0.0, 1.0, -1.0]], Np=3, Nu=3),
    # four players, player 2 borders everyone, players 3 and 4 symmetric
    "example4": dict(J=4, K=[[-1.0, 1.0, 0.0, 0.0], [1.0, -3.0, 1.0, 1.0], [0.0, 1.0, -2.0, 1.0],
                             [0.0, 1.0, 1.0, -2.0]], Np=3, Nu=3),
}

_SHARED = dict(beta=1.0, phi=1.0, A=0.5, c=0.5, rho=0.1, h=1e-3, P_max=0.7, U_max=0.5, tol=1e-6,
               max_iters=200_000)


def preset_spec(name: str, **overrides) -> GameSpec:
    """GameSpec of a named layout with GameSpec-field overrides (S/presets.py:44-57)."""
    if name not in _LAYOUTS:
        raise ValueError(f"unknown preset {name!r}; choose from {PRESET_NAMES}")
    params = {**_SHARED, **_LAYOUTS[name], **overrides}
    return GameSpec(**params)


def spec_to_dict(spec: GameSpec) -> dict:
    """JSON-ready dict of every GameSpec field (S/presets.py:60-77)."""
    out = {"J": spec.J, "K": np.asarray(spec.K).tolist()}
    for name in ("beta", "phi", "A", "c", "m"):
        out[name] = getattr(spec, name).tolist()
    out.update(rho=spec.rho, h=spec.h, P_max=spec.P_max, U_max=spec.U_max, Np=spec.Np.tolist(),
               Nu=spec.Nu.tolist(), tol=spec.tol, max_iters=spec.max_iters)
    return out


def spec_from_dict(data: dict) -> GameSpec:
    return GameSpec(**data)
