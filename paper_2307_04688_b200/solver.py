"""Collocation solver for the feedback equilibrium — drop-in mirror of ``chebnash.solver``
(S/solver.py) with every sweep on the B200.

Per sweep, one warp per (player, state node) binds the other players' controls in the drift
stacks, forms the Euler successors, evaluates the value interpolant there, fits the 1-D objective
and runs the safeguarded Newton maximiser (cb_solver.cu); the value interpolants are refitted by
the K1 transform.  `solve` keeps all fields on the device and runs sweeps back to back from CUDA
graphs with the stopping test on the device (cb_solve).  Block plans and worker counts are
accepted and validated exactly as in the reference but never change the result — every node's
arithmetic is fixed, so results are identical for every plan (the reference's contract,
S/solver.py:18-21).
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cheb1d import ChebBasis1D, CoefVector, make_basis, reference_nodes
from .chebnd import CoefTensor, TensorStack, stack_coeffs, tensor_coeffs
from .game import GameSpec, StateGrid, build_state_grid, dynamics, step

_CLAMP_WARN_FRACTION = 0.01  # S/solver.py:54

__all__ = [
    "BlockPlan", "partition", "ValueField", "PolicyField", "TimePath", "EquilibriumResult", "control_bases",
    "precompute_dynamics_stack", "newton_maximize", "bellman_sweep", "solve", "fit_policy", "simulate",
    "simulate_batch",
]


# ---------------------------------------------------------------------------------------------
# plan and result containers (S/solver.py:61-131)
# ---------------------------------------------------------------------------------------------

@dataclass(frozen=True)
class BlockPlan:
    """Exact factorisation N_b * N_f = N_P of the node count (S/solver.py:61-78)."""

    n_blocks: int
    block_size: int

    def __post_init__(self):
        if self.n_blocks < 1 or self.block_size < 1:
            raise ValueError("block counts must be positive")

    @property
    def n_nodes(self) -> int:
        return self.n_blocks * self.block_size

    def slices(self) -> list[slice]:
        f = self.block_size
        return [slice(k * f, (k + 1) * f) for k in range(self.n_blocks)]


def partition(n_nodes: int, n_blocks: int) -> BlockPlan:
    """n_nodes split into n_blocks contiguous blocks; n_blocks must divide (S/solver.py:81-87)."""
    if n_nodes < 1 or n_blocks < 1:
        raise ValueError("node and block counts must be positive")
    if n_nodes % n_blocks:
        raise ValueError(f"{n_blocks} does not divide {n_nodes} nodes")
    return BlockPlan(n_blocks=n_blocks, block_size=n_nodes // n_blocks)


@dataclass
class ValueField:
    """Per-player value node values (J, N_P) and state-space interpolants."""

    values: np.ndarray
    interpolants: list


@dataclass
class PolicyField:
    """Per-player control values on the state grid, (J, N_P)."""

    values: np.ndarray


@dataclass
class TimePath:
    """Simulated trajectory: times (T+1,), states and controls (T+1, J)."""

    t: np.ndarray
    states: np.ndarray
    controls: np.ndarray


@dataclass
class EquilibriumResult:
    """Outcome of the value iteration (S/solver.py:116-131)."""

    converged: bool
    iterations: int
    values: ValueField
    policy: PolicyField
    history: np.ndarray
    timings: dict
    clamp_fraction: float


# ---------------------------------------------------------------------------------------------
# offline precomputation
# ---------------------------------------------------------------------------------------------

def control_bases(spec: GameSpec) -> tuple[ChebBasis1D, ...]:
    """Per-player control bases on [0, U_max] with degrees spec.Nu (S/solver.py:136-138)."""
    return tuple(make_basis(int(n), 0.0, spec.U_max) for n in spec.Nu)


def precompute_dynamics_stack(spec: GameSpec, grid: StateGrid) -> list[TensorStack]:
    """Control-space drift interpolants, one stack member per state node (S/solver.py:141-159):
    member p of stack i interpolates u -> g_i(node_p, u) through all control node tuples.  The
    samples are the model's drift at those tuples; the transform runs on the GPU (stack_coeffs)."""
    bases = control_bases(spec)
    cshape = tuple(b.size for b in bases)
    mesh = np.meshgrid(*(b.nodes for b in bases), indexing="ij")
    controls = np.stack([m.ravel() for m in mesh], axis=-1)              # C-order control tuples
    vals = dynamics(spec, grid.nodes[None, :, :], controls[:, None, :])  # (n_controls, N_P, J)
    return [stack_coeffs(np.ascontiguousarray(vals[:, :, i].reshape(cshape + (grid.n_nodes,))), bases)
            for i in range(spec.J)]


# ---------------------------------------------------------------------------------------------
# device game record and buffers
# ---------------------------------------------------------------------------------------------

def _game_struct(spec: GameSpec, grid: StateGrid) -> _lib.CbGame:
    J = spec.J
    if J > _lib.MAX_PLAYERS:
        raise ValueError(f"at most {_lib.MAX_PLAYERS} players are supported on the device")
    if int(spec.Nu.max()) + 1 > _lib.MAX_CONTROL_NODES:
        raise ValueError(f"control degree above {_lib.MAX_CONTROL_NODES - 1} is not supported on the device")
    g = _lib.CbGame()
    g.J = J
    ub = control_bases(spec)
    for d in range(J):
        g.np[d] = grid.bases[d].size
        g.nu[d] = ub[d].size
        g.A[d] = float(spec.A[d])
        g.phi[d] = float(spec.phi[d])
        g.beta[d] = float(spec.beta[d])
        g.c[d] = float(spec.c[d])
        g.m[d] = float(spec.m[d])
        for e in range(J):
            g.K[d][e] = float(spec.K[d, e])
        rn = reference_nodes(int(spec.Nu[d]))
        for k in range(ub[d].size):
            g.unodes[d][k] = float(ub[d].nodes[k])
            g.rnodes[d][k] = float(rn[k])
    g.h, g.delta, g.P_max, g.U_max, g.tol = spec.h, spec.delta, spec.P_max, spec.U_max, spec.tol
    return g


class _Device:
    """Grid nodes + drift stacks resident on the device for one (spec, grid, stacks)."""

    def __init__(self, spec: GameSpec, grid: StateGrid, stacks):
        if len(stacks) != spec.J:
            raise ValueError("need one drift stack per player")
        for st in stacks:
            if st.count != grid.n_nodes:
                raise ValueError("drift stacks and grid disagree on the node count")
        t = _lib.require_cuda()
        self.spec, self.grid = spec, grid
        self.game = _game_struct(spec, grid)
        self.n = grid.n_nodes
        self.nodes = _lib.to_device(np.ascontiguousarray(grid.nodes))
        stk = t.cat([_lib.to_device(st.device_coefficients).reshape(-1) for st in stacks])
        lib = _lib.load()
        # node-major per-player drift tensors (the reference's _PlayerWork.coeffs), built once
        self.drift = _lib.empty((int(lib.cb_solver_drift_elems(ctypes.byref(self.game))),))
        _lib.check(lib.cb_solver_drift_layout(ctypes.byref(self.game), _lib.ptr(stk), _lib.ptr(self.drift),
                                              _lib.stream_handle()), "drift layout")
        # node values (J, N_P) read as (J, np_J, ..., np_1): the refit transform gives reversed-axis
        # coefficient tensors (no order="F" copy, S/solver.py:446)
        self.rev_shape = (spec.J,) + tuple(reversed(grid.shape))

    def refit(self, v_dev, coef_dev):
        rs = self.rev_shape
        _lib.check(_lib.load().cb_transform_axes(len(rs), _lib.i64_array(rs), 1, len(rs), _lib.ptr(v_dev),
                                                 _lib.ptr(coef_dev), None, 0, _lib.stream_handle()), "refit")

    def interpolants(self, coef_dev) -> list[CoefTensor]:
        """Reversed-axis device coefficients -> reference-order CoefTensors (S/solver.py:441-449)."""
        J = self.spec.J
        rs = tuple(reversed(self.grid.shape))
        out = []
        for i in range(J):
            c = coef_dev[i].reshape(rs).permute(*reversed(range(J))).contiguous()
            out.append(CoefTensor(self.grid.bases, c))
        return out


def _coef_arrays(values: ValueField, dev: _Device):
    """Current value interpolants -> reversed-axis device coefficients (J, N_P)."""
    t = _lib.require_cuda()
    J = dev.spec.J
    parts = []
    for i in range(J):
        c = values.interpolants[i]
        dense = c.dense_device() if isinstance(c, CoefTensor) else _lib.to_device(np.asarray(c, dtype=float))
        if tuple(dense.shape) != dev.grid.shape:
            raise ValueError("value interpolants and grid disagree on the shape")
        parts.append(dense.permute(*reversed(range(J))).contiguous().reshape(-1))
    return t.stack(parts)


# ---------------------------------------------------------------------------------------------
# maximiser (S/solver.py:326-356)
# ---------------------------------------------------------------------------------------------

def newton_maximize(coeffs: CoefVector, u0: float) -> tuple[float, float]:
    """Global maximiser of a 1-D interpolant over its interval: Newton point, both endpoints and
    the dense scan with bisection refinement (always evaluated here), on the GPU."""
    basis = coeffs.basis
    L = coeffs.coefficients.size
    if L > _lib.MAX_CONTROL_NODES:
        raise ValueError(f"degree above {_lib.MAX_CONTROL_NODES - 1} is not supported on the device")
    x0 = (2.0 * float(u0) - (basis.a + basis.b)) / (basis.b - basis.a)
    dc = _lib.to_device(coeffs.coefficients.reshape(1, -1))
    dx0 = _lib.to_device(np.array([x0]))
    x = _lib.empty((1,))
    f = _lib.empty((1,))
    _lib.check(_lib.load().cb_maximise_rows(1, L, _lib.ptr(dc), _lib.ptr(dx0), _lib.ptr(x), _lib.ptr(f), 1,
                                            _lib.stream_handle()), "newton_maximize")
    xv = float(_lib.to_host(x)[0])
    u = 0.5 * (basis.b - basis.a) * xv + 0.5 * (basis.a + basis.b)
    return u, float(_lib.to_host(f)[0])


def _maximise_rows(coef, x0, always_scan: bool = False):
    """Batched _maximise_block (S/solver.py:262-323) on the device: (m, L) rows -> (x, f)."""
    c = np.ascontiguousarray(coef, dtype=float)
    m, L = c.shape
    dc = _lib.to_device(c)
    dx0 = _lib.to_device(np.ascontiguousarray(x0, dtype=float))
    x = _lib.empty((m,))
    f = _lib.empty((m,))
    _lib.check(_lib.load().cb_maximise_rows(m, L, _lib.ptr(dc), _lib.ptr(dx0), _lib.ptr(x), _lib.ptr(f),
                                            1 if always_scan else 0, _lib.stream_handle()), "maximise")
    return _lib.to_host(x), _lib.to_host(f)


# ---------------------------------------------------------------------------------------------
# one sweep (S/solver.py:359-470)
# ---------------------------------------------------------------------------------------------

def bellman_sweep(spec: GameSpec, grid: StateGrid, values: ValueField, policy: PolicyField, stacks,
                  plan: BlockPlan | None = None) -> tuple[ValueField, PolicyField]:
    """One synchronous best-response sweep over all players and nodes, then the refit.  The plan is
    validated as in the reference; it never changes the result."""
    plan = plan if plan is not None else partition(grid.n_nodes, 1)
    if plan.n_nodes != grid.n_nodes:
        raise ValueError("block plan does not cover the grid")
    dev = _Device(spec, grid, stacks)
    t = _lib.require_cuda()
    J, n = spec.J, dev.n
    coef = _coef_arrays(values, dev)
    v = _lib.to_device(np.asarray(values.values, dtype=float).reshape(J, n))
    u = _lib.to_device(np.asarray(policy.values, dtype=float).reshape(J, n))
    v_out = _lib.empty((J, n))
    u_out = _lib.empty((J, n))
    clamped = t.zeros(1, dtype=t.int64, device=_lib.device())
    st = _lib.new_status()
    _lib.check(_lib.load().cb_bellman_sweep(ctypes.byref(dev.game), _lib.ptr(dev.nodes), _lib.ptr(dev.drift),
                                            _lib.ptr(coef), _lib.ptr(v), _lib.ptr(u), _lib.ptr(v_out),
                                            _lib.ptr(u_out), _lib.ptr(clamped), _lib.ptr(st), _lib.stream_handle()),
               "bellman_sweep")
    if _lib.read_status(st)[0]:
        raise FloatingPointError("non-finite objective sample in sweep")
    new_coef = _lib.empty((J, n))
    dev.refit(v_out, new_coef)
    vf = ValueField(values=_lib.to_host(v_out), interpolants=dev.interpolants(new_coef))
    return vf, PolicyField(values=_lib.to_host(u_out))


# ---------------------------------------------------------------------------------------------
# fixed-point driver (S/solver.py:477-570)
# ---------------------------------------------------------------------------------------------

def _initial_fields(spec: GameSpec, grid: StateGrid, init):
    n = grid.n_nodes
    if init is None:
        return np.zeros((spec.J, n)), np.broadcast_to(spec.A[:, None], (spec.J, n)).copy()
    values, policy = init
    v = np.array(getattr(values, "values", values), dtype=float)
    u = np.array(getattr(policy, "values", policy), dtype=float)
    if v.shape != (spec.J, n) or u.shape != (spec.J, n):
        raise ValueError(f"initial fields must have shape {(spec.J, n)}")
    if (u < 0.0).any() or (u > spec.U_max).any():
        raise ValueError("initial policy outside [0, U_max]")
    return v, u


def solve(spec: GameSpec, plan: BlockPlan | None = None, init=None, workers: int = 1) -> EquilibriumResult:
    """Iterate best-response sweeps until the per-player sup-norm value change drops below tol
    (S/solver.py:495-570), entirely on the device.  Non-convergence within max_iters is reported
    through `converged`, not raised."""
    t_start = time.perf_counter()
    grid = build_state_grid(spec)
    stacks = precompute_dynamics_stack(spec, grid)
    n = grid.n_nodes
    plan = plan if plan is not None else partition(n, 1)
    if plan.n_nodes != n:
        raise ValueError(f"block plan covers {plan.n_nodes} nodes, grid has {n}")
    if int(workers) < 1:
        raise ValueError("workers must be positive")
    v0, u0 = _initial_fields(spec, grid, init)
    if not np.isfinite(v0).all():  # the reference's initial _refit -> tensor_coeffs (S/chebnd.py:181-182)
        raise ValueError("samples must be finite")
    dev = _Device(spec, grid, stacks)
    t = _lib.require_cuda()
    J = spec.J
    v = _lib.empty((2, J, n))
    u = _lib.empty((2, J, n))
    coef = _lib.empty((2, J, n))
    v[0].copy_(_lib.to_device(v0))
    u[0].copy_(_lib.to_device(u0))
    max_iters = spec.max_iters
    lib = _lib.load()
    work = t.empty(int(lib.cb_solve_work_bytes(ctypes.byref(dev.game), max_iters)), dtype=t.uint8,
                   device=_lib.device())
    targets_per_sweep = n * sum(int(k) + 1 for k in spec.Nu) * J
    t_setup = time.perf_counter() - t_start
    iters = ctypes.c_int64(0)
    conv = ctypes.c_int(0)
    rc = lib.cb_solve(ctypes.byref(dev.game), _lib.ptr(dev.nodes), _lib.ptr(dev.drift), _lib.ptr(v), _lib.ptr(u),
                      _lib.ptr(coef), _lib.ptr(work), max_iters, ctypes.byref(iters), ctypes.byref(conv),
                      _lib.stream_handle())
    _lib.check(rc, "solve")
    it = int(iters.value)
    hist_bits = work[: max_iters * J * 8].view(t.float64).reshape(max_iters, J)[:it]
    clamps = work[max_iters * J * 8: max_iters * (J + 1) * 8].view(t.int64)[:it]
    fin = it % 2
    v_fin, u_fin = _lib.to_host(v[fin]), _lib.to_host(u[fin])
    history = _lib.to_host(hist_bits).reshape(-1, J)
    clamp_fraction = float(_lib.to_host(clamps).max() / targets_per_sweep) if it else 0.0
    if clamp_fraction > _CLAMP_WARN_FRACTION:
        warnings.warn(f"{clamp_fraction:.1%} of successor-state samples clamped to the state box; "
                      "P_max is probably too small", RuntimeWarning, stacklevel=2)
    t_total = time.perf_counter() - t_start
    return EquilibriumResult(
        converged=bool(conv.value), iterations=it,
        values=ValueField(values=v_fin, interpolants=dev.interpolants(coef[fin])),
        policy=PolicyField(values=u_fin), history=history,
        timings={"setup": t_setup, "sweeps": t_total - t_setup, "total": t_total},
        clamp_fraction=clamp_fraction)


# ---------------------------------------------------------------------------------------------
# trajectories (S/solver.py:577-629)
# ---------------------------------------------------------------------------------------------

def fit_policy(grid: StateGrid, policy: PolicyField) -> list[CoefTensor]:
    """State-space interpolants of the per-player policy node values (GPU build)."""
    shape = tuple(b.size for b in grid.bases)
    return [tensor_coeffs(np.asarray(policy.values[i]).reshape(shape, order="F"), grid.bases)
            for i in range(policy.values.shape[0])]


def _simulate_device(spec: GameSpec, policies, P0: np.ndarray, n_steps: int):
    J = spec.J
    if len(policies) != J:
        raise ValueError("need one policy interpolant per player")
    grid = build_state_grid(spec)
    for pol in policies:
        if tuple(pol.shape) != grid.shape:
            raise ValueError("policy interpolants and the state grid disagree on the shape")
    t = _lib.require_cuda()
    game = _game_struct(spec, grid)
    pols = t.cat([pol.dense_device().reshape(-1) for pol in policies])
    B = P0.shape[0]
    dp0 = _lib.to_device(np.ascontiguousarray(P0, dtype=float))
    states = _lib.empty((B, n_steps + 1, J))
    controls = _lib.empty((B, n_steps + 1, J))
    _lib.check(_lib.load().cb_simulate(ctypes.byref(game), B, _lib.ptr(pols), _lib.ptr(dp0), n_steps,
                                       _lib.ptr(states), _lib.ptr(controls), _lib.stream_handle()), "simulate")
    return _lib.to_host(states), _lib.to_host(controls)


def simulate(spec: GameSpec, policies, p0, n_steps: int) -> TimePath:
    """Closed-loop rollout u_n = clip(policy(p_n)), Euler step, repeat (S/solver.py:597-629); the
    whole trajectory runs in one kernel (cb_simulate)."""
    J = spec.J
    if len(policies) != J:
        raise ValueError("need one policy interpolant per player")
    p = np.asarray(p0, dtype=float).copy()
    if p.shape != (J,) or (p < 0.0).any() or (p > spec.P_max).any():
        raise ValueError(f"p0 must lie in [0, {spec.P_max}]^{J}")
    n_steps = int(n_steps)
    states, controls = _simulate_device(spec, policies, p.reshape(1, J), n_steps)
    return TimePath(t=np.arange(n_steps + 1) * spec.h, states=states[0], controls=controls[0])


def simulate_batch(spec: GameSpec, policies, p0s, n_steps: int) -> tuple[np.ndarray, np.ndarray]:
    """Batched form of `simulate`: B initial states (B, J) -> states and controls
    (B, n_steps + 1, J), one warp per trajectory."""
    P0 = np.asarray(p0s, dtype=float)
    if P0.ndim != 2 or P0.shape[1] != spec.J or (P0 < 0.0).any() or (P0 > spec.P_max).any():
        raise ValueError(f"initial states must be (B, {spec.J}) inside [0, {spec.P_max}]")
    return _simulate_device(spec, policies, P0, int(n_steps))
