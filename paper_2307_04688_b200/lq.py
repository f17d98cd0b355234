"""Closed-form linear-feedback equilibrium of the LQ game — the reference's validation oracle
(S/oracle.py), with the coefficient-space fixed point iterated on the GPU (cb_lq).

For the linear-quadratic game the discounted Bellman operator maps quadratic values
V_i(p) = p'Q_i p + b_i'p + d_i and affine feedback u_i(p) = max(0, e_i + f_i'p) into the same
family while the emission constraint is inactive, so iterating that exact update converges to the
equilibrium without any interpolation.  `policy_error` compares a collocation policy against it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cheb1d import _freeze
from .game import GameSpec, StateGrid, build_state_grid

_COEF_TOL = 1e-13          # S/oracle.py:25
_MAX_ITERS = 1_000_000     # :26

__all__ = ["LQFeedback", "lq_bellman_update", "lq_solve", "policy_error"]


@dataclass(frozen=True)
class LQFeedback:
    """Quadratic value coefficients and affine feedback per player (S/oracle.py:31-57)."""

    Q: np.ndarray
    b: np.ndarray
    d: np.ndarray
    e: np.ndarray
    f: np.ndarray
    iterations: int
    negative_fraction: float
    high_fraction: float

    def __post_init__(self):
        for name in ("Q", "b", "d", "e", "f"):
            object.__setattr__(self, name, _freeze(np.array(getattr(self, name), dtype=float)))

    def policy(self, states) -> np.ndarray:
        """Feedback controls max(0, e_i + f_i p) at states (..., J)."""
        p = np.asarray(states, dtype=float)
        return np.maximum(0.0, self.e + p @ self.f.T)

    def value(self, states) -> np.ndarray:
        """Quadratic values p'Q_i p + b_i'p + d_i at states (..., J)."""
        p = np.asarray(states, dtype=float)
        return np.einsum("...a,iab,...b->...i", p, self.Q, p) + p @ self.b.T + self.d


def _game(spec: GameSpec):
    from .solver import _game_struct

    return _game_struct(spec, build_state_grid(spec))


def _pack(J, Q, b, d, e, f) -> np.ndarray:
    return np.concatenate([np.asarray(Q, float).reshape(-1), np.asarray(b, float).reshape(-1),
                           np.asarray(d, float).reshape(-1), np.asarray(e, float).reshape(-1),
                           np.asarray(f, float).reshape(-1)])


def _unpack(J, v):
    nQ, nb = J ** 3, J * J
    Q = v[:nQ].reshape(J, J, J)
    b = v[nQ:nQ + nb].reshape(J, J)
    d = v[nQ + nb:nQ + nb + J]
    e = v[nQ + nb + J:nQ + nb + 2 * J]
    f = v[nQ + nb + 2 * J:].reshape(J, J)
    return Q, b, d, e, f


def _run(spec: GameSpec, state: np.ndarray, mode: int, max_iters: int):
    J = spec.J
    t = _lib.require_cuda()
    g = _game(spec)
    dstate = _lib.to_device(state)
    work = _lib.empty((state.size + 2,))
    its = ctypes.c_int64(0)
    _lib.check(_lib.load().cb_lq(ctypes.byref(g), _lib.ptr(dstate), _lib.ptr(work), int(max_iters), _COEF_TOL, mode,
                                 ctypes.byref(its), _lib.stream_handle()), "lq")
    del t
    return _unpack(J, _lib.to_host(dstate)), int(its.value)


def lq_bellman_update(spec: GameSpec, Q, b, d, e, f) -> tuple[np.ndarray, ...]:
    """One exact simultaneous best-response update of every player's quadratic data
    (S/oracle.py:65-109): interior maximisation in closed form, then
    V_i'(p) = delta (h G_i(p_i, u_i*(p)) + V_i(next state))."""
    J = spec.J
    (Qn, bn, dn, en, fn), _ = _run(spec, _pack(J, Q, b, d, e, f), 0, 1)
    return Qn, bn, dn, en, fn


def lq_solve(spec: GameSpec, grid: StateGrid | None = None) -> LQFeedback:
    """Equilibrium of the unconstrained LQ game (S/oracle.py:112-163): the update iterated from the
    zero value function until (Q, b, e, f) are stationary, the constant term closed from its scalar
    fixed point; records where the unconstrained feedback leaves [0, U_max] on the grid."""
    J = spec.J
    (Q, b, d, e, f), its = _run(spec, np.zeros(J ** 3 + 2 * J * J + 2 * J), 1, _MAX_ITERS)
    if grid is None:
        grid = build_state_grid(spec)
    raw = e + grid.nodes @ f.T
    return LQFeedback(Q=Q, b=b, d=d, e=e, f=f, iterations=its,
                      negative_fraction=float(np.mean(np.any(raw < 0.0, axis=1))),
                      high_fraction=float(np.mean(np.any(raw > spec.U_max, axis=1))))


def policy_error(policy_values, feedback: LQFeedback, grid: StateGrid) -> float:
    """(1/N) sqrt(sum over nodes and players of the squared policy gap) (S/oracle.py:166-195); refused
    where the oracle's unconstrained feedback leaves [0, U_max] on the grid."""
    values = np.asarray(getattr(policy_values, "values", policy_values), dtype=float)
    J = feedback.e.size
    if values.shape != (J, grid.n_nodes):
        raise ValueError(f"expected policy of shape {(J, grid.n_nodes)}, got {values.shape}")
    if feedback.negative_fraction > 0.0:
        raise ValueError("oracle invalid: unconstrained feedback is negative on "
                         f"{feedback.negative_fraction:.1%} of grid nodes")
    if feedback.high_fraction > 0.0:
        raise ValueError("oracle invalid: unconstrained feedback exceeds U_max on "
                         f"{feedback.high_fraction:.1%} of grid nodes")
    reference = feedback.policy(grid.nodes).T
    return float(np.sqrt(np.sum((values - reference) ** 2)) / grid.n_nodes)
