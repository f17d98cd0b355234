"""Time-stepping loop (K4) — the solver skeleton of S/solver.py:541-550 (sweep, refit, repeat)
specialised to the BASELINE loop configs 3 / 5b: fixed linear drift g(x) = A x, so one step is

    C   = tensor_coeffs(V_t)                                     (S/solver.py:441-449, _refit)
    y_i = clip(x_i + dt * A x_i, box)                            (S/solver.py:383-386)
    V_{t+1}(x_i) = V_t-interpolant(y_i) - dt * |x_i|^2           (S/solver.py:388-397)

over all grid nodes x_i.  On one GPU the whole loop is device resident (cb_advect_loop, CUDA graph
of the build + evaluate pair, no host round trips).  Across GPUs the nodes are sharded in
contiguous slabs and the node values are all-gathered once per step (dist.py).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _box(bases):
    lo = [float(b.a) for b in bases]
    hi = [float(b.b) for b in bases]
    return lo, hi


def advect_loop(values, bases, A, dt: float, steps: int, use_graph: bool = True):
    """Run `steps` steps of V <- V(clip(x + dt A x)) - dt|x|^2 on the node grid of `bases`.

    values: (n_1, ..., n_J) node values in C order (numpy or CUDA tensor).  Returns the same kind.
    Raises ValueError("samples must be finite") if a non-finite value appears (the reference's
    tensor_coeffs check, S/chebnd.py:181-185)."""
    bases = tuple(bases)
    shape = tuple(b.size for b in bases)
    is_t = _lib.torch().is_tensor(values)
    v_shape = tuple(values.shape) if is_t else np.shape(values)
    if tuple(v_shape) != shape:
        raise ValueError(f"sample shape {tuple(v_shape)} does not match bases {shape}")
    J = len(shape)
    A = np.asarray(A, dtype=float)
    if A.shape != (J, J):
        raise ValueError(f"drift matrix must be {J}x{J}")
    if steps < 0:
        raise ValueError("steps must be non-negative")
    dv = _lib.to_device(values).clone()
    tmp = _lib.empty(shape)
    L = _lib.eval_layout(shape)
    coef = _lib.empty((L["elems"],))
    st = _lib.new_status()
    lo, hi = _box(bases)
    _lib.check(
        _lib.load().cb_advect_loop(J, _lib.i64_array(shape), _lib.ptr(dv), _lib.ptr(tmp), _lib.ptr(coef), int(steps),
                                   _lib.dbl_array(A), float(dt), _lib.dbl_array(lo), _lib.dbl_array(hi), _lib.ptr(st),
                                   1 if use_graph else 0, _lib.stream_handle()),
        "advect_loop",
    )
    _lib.raise_for_samples(st)
    return dv if is_t else _lib.to_host(dv)


class CudaStepBackend:
    """Device kernels behind one sharded step: replicated build + slab evaluation."""

    def __init__(self, bases, A, dt):
        self.bases = tuple(bases)
        self.shape = tuple(b.size for b in self.bases)
        self.J = len(self.shape)
        self.A = _lib.dbl_array(np.asarray(A, dtype=float))
        self.dt = float(dt)
        lo, hi = _box(self.bases)
        self.lo, self.hi = _lib.dbl_array(lo), _lib.dbl_array(hi)
        self.sizes = _lib.i64_array(self.shape)
        self.L = _lib.eval_layout(self.shape)
        self.coef = _lib.empty((self.L["elems"],))
        self.status = _lib.new_status()

    def zeros(self, n):
        t = _lib.require_cuda()
        return t.zeros(int(n), dtype=t.float64, device=_lib.device())

    def to_buffer(self, values):
        return _lib.to_device(values).reshape(-1)

    def build(self, full_values):
        _lib.check(_lib.load().cb_tensor_coeffs(self.J, self.sizes, _lib.ptr(full_values), _lib.ptr(self.coef),
                                                _lib.ptr(self.status), _lib.stream_handle()), "build")

    def eval_slab(self, begin: int, count: int, out_view):
        if count <= 0:
            return
        _lib.check(_lib.load().cb_eval_advected(self.J, self.sizes, _lib.ptr(self.coef), int(begin), int(count), self.A,
                                                self.dt, self.lo, self.hi, 1, _lib.ptr(out_view), _lib.stream_handle()),
                   "eval_slab")

    def finish(self, full_values):
        _lib.raise_for_samples(self.status)
        return full_values

    # --- fused exchange (dist.PeerShardedAdvectLoop) ---
    def exchange_buffers(self, bufs, group=None):
        """CUDA-IPC map every rank's node-value buffers: returns dests[b][r] = device address of
        rank r's buffer b in this process (own buffers unmapped)."""
        import torch.distributed as dist

        lib = _lib.load()
        self._mapped = []
        recs = []
        for b in bufs:
            rec = ctypes.create_string_buffer(72)
            _lib.check(lib.cb_ipc_export(_lib.ptr(b), rec), "ipc_export")
            recs.append(rec.raw)
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        allrecs = [recs]
        if world > 1:
            allrecs = [None] * world
            dist.all_gather_object(allrecs, recs, group=group)
        dests = [[0] * world for _ in bufs]
        for r in range(world):
            for i, b in enumerate(bufs):
                if r == rank:
                    dests[i][r] = _lib.ptr(b)
                    continue
                p, base = ctypes.c_void_p(), ctypes.c_void_p()
                _lib.check(lib.cb_ipc_import(allrecs[r][i], ctypes.byref(p), ctypes.byref(base)), "ipc_import")
                self._mapped.append(base.value)
                dests[i][r] = p.value
        t = _lib.require_cuda()
        self._flag = t.zeros(1, dtype=t.float64, device=_lib.device())
        return dests

    def eval_slab_peers(self, begin: int, count: int, dests):
        if count <= 0:
            return
        arr = (ctypes.c_void_p * len(dests))(*dests)
        _lib.check(_lib.load().cb_eval_advected_peers(self.J, self.sizes, _lib.ptr(self.coef), int(begin), int(count),
                                                      self.A, self.dt, self.lo, self.hi, 1, arr, len(dests),
                                                      _lib.stream_handle()),
                   "eval_slab_peers")

    def barrier(self, group=None):
        """Orders every rank's peer stores of this step before any rank's next build: a 1-element
        NCCL all-reduce on the compute stream (host-asynchronous); under gloo (several ranks sharing
        one GPU in the tests) a device synchronize + host barrier."""
        import torch.distributed as dist

        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(self._flag, group=group)
        else:
            _lib.require_cuda().cuda.synchronize()
            dist.barrier(group=group)

    def close_buffers(self):
        for base in getattr(self, "_mapped", []):
            _lib.load().cb_ipc_close(base)
        self._mapped = []
