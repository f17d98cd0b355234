"""CPU oracle for the Bellman sweep / `solve` of the reference solver — TEST INFRASTRUCTURE ONLY.

Same rules as oracle/cheb_oracle.py: only tests/, __graft_entry__.smoke() and bench.py's CPU legs
may import it; the product package never does.  It restates in numpy the collocation solver of
``chebnash`` 0.1.0 (S/solver.py, S/game.py, S/presets.py), SURVEY.md §8f row 1:

* the game (drift g, stage payoff, Euler step)                 S/game.py:140-189
* the state grid (dim-1-fastest node enumeration)              S/game.py:117-126
* the control-space drift stacks                               S/solver.py:134-159
* per-player constants (bind order, B0, M0, stage table)       S/solver.py:162-198
* one block best response (bind, drift, successor, value,
  objective, 1-D fit, safeguarded Newton maximiser)            S/solver.py:226-409
* refit, sweep, fixed-point driver                             S/solver.py:412-570
* fit_policy / simulate                                        S/solver.py:577-629

Parity of this restatement is PINNED by tests/test_oracle_solver.py against
tests/golden/golden_solver_v1.npz, which tests/golden/make_golden_solver.py produced by running the
reference solver itself.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .cheb_oracle import (
    cheb_transform,
    derivative_array,
    eval_points,
    interval_nodes,
    reference_nodes,
    row_basis,
    tensor_coeffs,
)

NEWTON_MAX_ITER = 30      # S/solver.py:50
NEWTON_TOL = 1e-12        # :51
SCAN_POINTS = 257         # :52
BISECT_STEPS = 60         # :53
CLAMP_WARN_FRACTION = 0.01  # :54


# ---------------------------------------------------------------------------------------------
# game model (plain parameter record; validation lives in the product's GameSpec)
# ---------------------------------------------------------------------------------------------

@dataclass
class Game:
    J: int
    K: np.ndarray
    beta: np.ndarray
    phi: np.ndarray
    A: np.ndarray
    c: np.ndarray
    m: np.ndarray
    rho: float
    h: float
    P_max: float
    U_max: float
    Np: np.ndarray
    Nu: np.ndarray
    tol: float
    max_iters: int

    @property
    def delta(self) -> float:
        return 1.0 - self.rho * self.h


def game_from_golden(g, key: str) -> Game:
    sc = g[f"{key}_spec_scalars"]
    return Game(J=int(sc[0]), K=g[f"{key}_spec_K"], beta=g[f"{key}_spec_beta"], phi=g[f"{key}_spec_phi"],
                A=g[f"{key}_spec_A"], c=g[f"{key}_spec_c"], m=g[f"{key}_spec_m"], rho=float(sc[1]),
                h=float(sc[2]), P_max=float(sc[3]), U_max=float(sc[4]), Np=g[f"{key}_spec_Np"].astype(int),
                Nu=g[f"{key}_spec_Nu"].astype(int), tol=float(sc[5]), max_iters=int(sc[6]))


def drift(game: Game, p, u) -> np.ndarray:
    """g_i = (sum_j k_ij p_j - p_i sum_j k_ij)/m_i - c_i p_i + beta_i u_i  (S/game.py:140-151)."""
    p = np.asarray(p, dtype=float)
    u = np.asarray(u, dtype=float)
    exch = p @ np.asarray(game.K).T - p * np.asarray(game.K).sum(axis=1)
    return exch / game.m - game.c * p + game.beta * u


def euler_step(game: Game, p, u) -> np.ndarray:
    """p + h g(p, u), clipped to [0, P_max] (S/game.py:165-168)."""
    return np.clip(np.asarray(p, dtype=float) + game.h * drift(game, p, u), 0.0, game.P_max)


def grid_nodes(game: Game) -> np.ndarray:
    """(N_P, J) state nodes, dimension 1 fastest (S/game.py:117-126)."""
    axes = [interval_nodes(int(n), 0.0, game.P_max) for n in game.Np]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel(order="F") for m in mesh], axis=-1)


def drift_stacks(game: Game, nodes: np.ndarray) -> list[np.ndarray]:
    """Per component i: (Nu_1+1, ..., Nu_J+1, N_P) control-space coefficients of u -> g_i(node, u)
    (S/solver.py:134-159): samples at the control node tuples, transformed along the control axes."""
    J = game.J
    axes = [interval_nodes(int(n), 0.0, game.U_max) for n in game.Nu]
    cshape = tuple(a.size for a in axes)
    mesh = np.meshgrid(*axes, indexing="ij")
    out = []
    for i in range(J):
        # samples[l_1..l_J, p] = g_i(node_p, (u_{l_1}, ..., u_{l_J}))
        U = np.stack([m for m in mesh], axis=-1)                      # cshape + (J,)
        g = drift(game, nodes[None, :, :], U.reshape(-1, J)[:, None, :])[:, :, i]
        s = g.reshape(cshape + (nodes.shape[0],))
        for ax in range(J):
            s = np.moveaxis(cheb_transform(s, 0), 0, J - 1)          # stack_coeffs order
        out.append(np.ascontiguousarray(s))
    return out


def transform_matrix(degree: int) -> np.ndarray:
    """diag(s) B(ref nodes)^T diag(w) (S/solver.py:162-171)."""
    size = degree + 1
    B = row_basis(reference_nodes(degree), size)
    w = np.ones(size)
    w[[0, -1]] = 0.5
    s = np.full(size, 2.0 / degree)
    s[[0, -1]] = 1.0 / degree
    return s[:, None] * B.T * w[None, :]


class Player:
    """Per-player constants (S/solver.py:174-198)."""

    def __init__(self, game: Game, nodes: np.ndarray, stacks: list[np.ndarray], i: int):
        J = game.J
        self.i = i
        self.others = [j for j in range(J) if j != i]
        self.other_sizes = [int(game.Nu[j]) + 1 for j in self.others]
        perm = [0] + [1 + j for j in self.others] + [1 + i]
        self.coeffs = np.ascontiguousarray(
            np.stack([np.transpose(np.moveaxis(st, -1, 0), perm) for st in stacks], axis=-1))
        self.K = int(game.Nu[i]) + 1
        self.B0 = row_basis(reference_nodes(int(game.Nu[i])), self.K)
        self.M0 = transform_matrix(int(game.Nu[i]))
        un = interval_nodes(int(game.Nu[i]), 0.0, game.U_max)
        self.stage = game.h * ((un * (game.A[i] - 0.5 * un))[None, :] - (0.5 * game.phi[i] * nodes[:, i] ** 2)[:, None])


# ---------------------------------------------------------------------------------------------
# safeguarded maximiser (S/solver.py:226-356)
# ---------------------------------------------------------------------------------------------

def clenshaw_rows(c: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Rows of (m, L) coefficients at points (m,) (S/solver.py:226-236)."""
    L = c.shape[1]
    if L == 1:
        return c[:, 0].copy()
    x2 = 2.0 * x
    b1 = np.zeros_like(x)
    b2 = np.zeros_like(x)
    for k in range(L - 1, 0, -1):
        b1, b2 = c[:, k] + x2 * b1 - b2, b1
    return c[:, 0] + x * b1 - b2


def scan_refine(coef: np.ndarray, q1: np.ndarray):
    """257-point scan + 60 bisection steps on f' (S/solver.py:239-259)."""
    m = coef.shape[0]
    xs = np.linspace(-1.0, 1.0, SCAN_POINTS)
    vals = np.stack([clenshaw_rows(coef, np.full(m, x)) for x in xs], axis=1)
    k = np.argmax(vals, axis=1)
    x_scan = xs[k]
    lo = xs[np.maximum(k - 1, 0)]
    hi = xs[np.minimum(k + 1, SCAN_POINTS - 1)]
    s_lo = np.sign(clenshaw_rows(q1, lo))
    for _ in range(BISECT_STEPS):
        mid = 0.5 * (lo + hi)
        same = np.sign(clenshaw_rows(q1, mid)) == s_lo
        lo, hi = np.where(same, mid, lo), np.where(same, hi, mid)
    x_ref = 0.5 * (lo + hi)
    keep_ref = clenshaw_rows(coef, x_ref) >= vals[np.arange(m), k]
    return np.where(keep_ref, x_ref, x_scan), x_scan


def maximise_rows(coef: np.ndarray, x0: np.ndarray, always_scan: bool = False):
    """Projected Newton on f' from the warm start, endpoints, scan fallback (S/solver.py:262-323)."""
    m, L = coef.shape
    sign = np.where(np.arange(L) % 2 == 0, 1.0, -1.0)
    f_hi = coef.sum(axis=1)
    f_lo = (coef * sign).sum(axis=1)
    if L <= 2:
        return np.where(f_hi >= f_lo, 1.0, -1.0), np.maximum(f_hi, f_lo)
    q1 = derivative_array(coef)
    q2 = derivative_array(q1)
    x = np.clip(np.asarray(x0, dtype=float), -1.0, 1.0).copy()
    moving = np.ones(m, dtype=bool)
    failed = np.zeros(m, dtype=bool)
    for _ in range(NEWTON_MAX_ITER):
        d1 = clenshaw_rows(q1, x)
        d2 = clenshaw_rows(q2, x)
        flat = np.abs(d2) <= 1e-300
        raw = x - d1 / np.where(flat, 1.0, d2)
        xn = np.clip(raw, -1.0, 1.0)
        failed |= (moving & ~flat & (raw != xn)) | (moving & flat)
        moving &= ~flat
        step = np.abs(xn - x)
        x = np.where(moving, xn, x)
        moving &= step > NEWTON_TOL
        if not moving.any():
            break
    failed |= moving
    failed |= clenshaw_rows(q2, x) >= 0.0
    if always_scan:
        failed[:] = True
    best_x = x.copy()
    best_f = clenshaw_rows(coef, x)
    for cx, cf in ((-1.0, f_lo), (1.0, f_hi)):
        up = cf > best_f
        best_x = np.where(up, cx, best_x)
        best_f = np.where(up, cf, best_f)
    if failed.any():
        idx = np.flatnonzero(failed)
        x_fb, x_scan = scan_refine(coef[idx], q1[idx])
        for cx in (x_fb, x_scan):
            cf = clenshaw_rows(coef[idx], cx)
            up = cf > best_f[idx]
            best_x[idx[up]] = cx[up]
            best_f[idx[up]] = cf[up]
    return best_x, best_f


def newton_maximize(coef: np.ndarray, a: float, b: float, u0: float):
    """(u*, value) of a 1-D interpolant on [a, b] (S/solver.py:326-356)."""
    x0 = (2.0 * u0 - (a + b)) / (b - a)
    x, f = maximise_rows(np.asarray(coef, dtype=float)[None, :], np.array([x0]), always_scan=True)
    return 0.5 * (b - a) * float(x[0]) + 0.5 * (a + b), float(f[0])


# ---------------------------------------------------------------------------------------------
# sweep and driver
# ---------------------------------------------------------------------------------------------

class Solver:
    def __init__(self, game: Game):
        self.game = game
        self.nodes = grid_nodes(game)
        self.shape = tuple(int(n) + 1 for n in game.Np)
        self.stacks = drift_stacks(game, self.nodes)
        self.players = [Player(game, self.nodes, self.stacks, i) for i in range(game.J)]

    def refit(self, values: np.ndarray) -> list[np.ndarray]:
        """Per-player coefficient tensors of the node values (order-F reshape, S/solver.py:441-449)."""
        return [tensor_coeffs(values[i].reshape(self.shape, order="F")) for i in range(self.game.J)]

    def best_response(self, i: int, coefs: list[np.ndarray], policy: np.ndarray, sl: slice = slice(None)):
        """Player i on the node block `sl` (_best_response_block, S/solver.py:359-409); returns
        (u, v, clamped count) for the block."""
        g = self.game
        pw = self.players[i]
        nodes = self.nodes[sl]
        n = nodes.shape[0]
        cur = pw.coeffs[sl]
        for j, size in zip(pw.others, pw.other_sizes):
            Bj = row_basis(policy[j, sl] * (2.0 / g.U_max) - 1.0, size)         # (n, size)
            cur = np.einsum("pl,plr->pr", Bj, cur.reshape(n, size, -1))
        dr = np.einsum("kl,plc->pkc", pw.B0, cur.reshape(n, pw.K, g.J))     # drift at own nodes
        succ = nodes[:, None, :] + g.h * dr
        clipped = np.clip(succ, 0.0, g.P_max)
        clamped = int(np.count_nonzero(clipped != succ))
        pts = clipped.reshape(-1, g.J) * (2.0 / g.P_max) - 1.0
        v_next = eval_points(coefs[i], pts).reshape(n, pw.K)
        obj = g.delta * (pw.stage[sl] + v_next)
        if not np.isfinite(obj).all():
            raise FloatingPointError("non-finite objective sample in sweep")
        fit = obj @ pw.M0.T
        x, f = maximise_rows(fit, policy[i, sl] * (2.0 / g.U_max) - 1.0)
        return (x + 1.0) * (0.5 * g.U_max), f, clamped

    def sweep(self, coefs, policy, executor=None, blocks: int = 1):
        """One sweep over (player, node block) tasks (_run_sweep, S/solver.py:412-438): serial, or
        on a ThreadPoolExecutor with disjoint writes when `executor` is given."""
        J = self.game.J
        n = self.nodes.shape[0]
        u = np.empty((J, n))
        v = np.empty((J, n))
        size = -(-n // max(1, blocks))
        tasks = [(i, slice(a, min(n, a + size))) for i in range(J) for a in range(0, n, size)]

        def run(t):
            i, sl = t
            u[i, sl], v[i, sl], c = self.best_response(i, coefs, policy, sl)
            return c

        counts = list(executor.map(run, tasks)) if executor is not None else [run(t) for t in tasks]
        return u, v, int(sum(counts))

    def solve(self, values=None, policy=None, max_iters: int | None = None, workers: int = 1, blocks: int = 1):
        """Fixed-point driver (S/solver.py:495-570): returns dict of the EquilibriumResult fields."""
        g = self.game
        n = self.nodes.shape[0]
        v = np.zeros((g.J, n)) if values is None else np.array(values, dtype=float)
        u = np.broadcast_to(np.asarray(g.A)[:, None], (g.J, n)).copy() if policy is None else np.array(policy)
        coefs = self.refit(v)
        targets = n * sum(p.K for p in self.players) * g.J
        hist, clamp_frac, converged, it = [], 0.0, False, 0
        ex = None
        if workers > 1:
            from concurrent.futures import ThreadPoolExecutor

            ex = ThreadPoolExecutor(max_workers=workers)
        for it in range(1, (max_iters or g.max_iters) + 1):
            u_new, v_new, cl = self.sweep(coefs, u, ex, blocks)
            clamp_frac = max(clamp_frac, cl / targets)
            d = np.max(np.abs(v_new - v), axis=1)
            hist.append(d)
            v, u = v_new, u_new
            coefs = self.refit(v)
            if float(d.max()) < g.tol:
                converged = True
                break
        if ex is not None:
            ex.shutdown()
        return dict(converged=converged, iterations=it, values=v, policy=u, coefs=coefs,
                    history=np.array(hist).reshape(-1, g.J), clamp_fraction=clamp_frac)


def simulate(game: Game, policy_coefs: list[np.ndarray], p0, n_steps: int):
    """Closed-loop Euler rollout with clipped controls (S/solver.py:597-629)."""
    J = game.J
    p = np.asarray(p0, dtype=float).copy()
    states = np.empty((n_steps + 1, J))
    controls = np.empty((n_steps + 1, J))
    for t in range(n_steps + 1):
        states[t] = p
        x = p * (2.0 / game.P_max) - 1.0
        u = np.array([eval_points(c, x[None, :])[0] for c in policy_coefs])
        u = np.clip(u, 0.0, game.U_max)
        controls[t] = u
        if t < n_steps:
            p = euler_step(game, p, u)
    return states, controls


def discounted_payoff(game: Game, states, controls, horizon: int) -> np.ndarray:
    """h sum_{n=1}^{H} delta^n G_i(u_n, p_n) (S/game.py:171-189)."""
    if horizon == 0:
        return np.zeros(game.J)
    ps, us = states[1:horizon + 1], controls[1:horizon + 1]
    gains = us * (game.A - 0.5 * us) - 0.5 * game.phi * ps ** 2
    return game.h * (game.delta ** np.arange(1, horizon + 1) @ gains)
