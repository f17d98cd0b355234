"""Tensor-product Chebyshev interpolation in J dimensions — drop-in mirror of ``chebnash.chebnd``
(reference: pkg/src/chebnash/chebnd.py, cited S/chebnd.py:<line>) on the B200.

Containers keep the reference's constructor / attribute surface (``bases``, ``coefficients``,
``ndim``, ``count``, ``member``) but hold their coefficients in GPU memory: a ``CoefTensor``
keeps the eval layout consumed by the DMMA evaluator (include/chebnash_b200.h), a
``TensorStack`` the dense (n_1..n_J, N_P) array.  ``.coefficients`` returns a read-only numpy
array (copied back once, lazily), so code written against the reference keeps working, while
chained GPU calls (build -> evaluate) never leave the device.

Public functions take array-likes (numpy in -> numpy out, as in the reference) or CUDA torch
tensors (tensor in -> tensor out, no host round trip).  Every numeric step runs in
libchebnash_b200.so; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cheb1d import ChebBasis1D, _freeze

__all__ = [
    "CoefTensor",
    "TensorStack",
    "GatherIndex",
    "basis_matrix",
    "tensor_coeffs",
    "stack_coeffs",
    "eval_axis",
    "make_gather_index",
    "eval_diagonal_batch",
    "eval_full",
    "eval_points",
    "eval_grid",
]


def _is_tensor(x) -> bool:
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


class _Frozen:
    """Assignment guard mirroring the reference's frozen dataclasses."""

    __slots__ = ()

    def __setattr__(self, name, value):
        raise dataclasses.FrozenInstanceError(f"cannot assign to field '{name}'")

    def __delattr__(self, name):
        raise dataclasses.FrozenInstanceError(f"cannot delete field '{name}'")


def _set(obj, name, value):
    object.__setattr__(obj, name, value)


class CoefTensor(_Frozen):
    """Coefficients of one J-mode tensor-product interpolant (S/chebnd.py:33-54).

    ``coefficients[l1, ..., lJ]`` multiplies T_l1(x_1) ... T_lJ(x_J).  Device storage: the eval
    layout (rows = leading modes, columns = trailing modes, zero padded)."""

    __slots__ = ("bases", "_host", "_dev")

    def __init__(self, bases, coefficients):
        bases = tuple(bases)
        shape = tuple(b.size for b in bases)
        if _is_tensor(coefficients):
            dense = _lib.to_device(coefficients)
            if tuple(dense.shape) != shape:
                raise ValueError(f"coefficient shape {tuple(dense.shape)} does not match bases {shape}")
            _set(self, "bases", bases)
            _set(self, "_host", None)
            _set(self, "_dev", _pack(shape, dense))
            return
        coef = np.array(coefficients, dtype=float, order="C", copy=True)
        if coef.shape != shape:
            raise ValueError(f"coefficient shape {coef.shape} does not match bases {shape}")
        _set(self, "bases", bases)
        _set(self, "_host", _freeze(coef))
        _set(self, "_dev", None)

    @classmethod
    def _from_eval_layout(cls, bases, dev) -> "CoefTensor":
        obj = cls.__new__(cls)
        _set(obj, "bases", tuple(bases))
        _set(obj, "_host", None)
        _set(obj, "_dev", dev)
        return obj

    @property
    def shape(self) -> tuple:
        return tuple(b.size for b in self.bases)

    @property
    def ndim(self) -> int:
        return len(self.bases)

    @property
    def coefficients(self) -> np.ndarray:
        if self._host is None:
            dense = _unpack(self.shape, self._dev)
            _set(self, "_host", _freeze(_lib.to_host(dense)))
        return self._host

    @property
    def device_coefficients(self):
        """Eval-layout CUDA tensor (flat, R8*Kp doubles)."""
        if self._dev is None:
            _set(self, "_dev", _pack(self.shape, _lib.to_device(self._host)))
        return self._dev

    def dense_device(self):
        """Dense C-order CUDA tensor of the coefficients."""
        return _unpack(self.shape, self.device_coefficients)

    def __repr__(self):
        return f"CoefTensor(bases={self.bases!r})"


class TensorStack(_Frozen):
    """N_P interpolants with a shared layout, stacked on the trailing axis (S/chebnd.py:57-81)."""

    __slots__ = ("bases", "_host", "_dev")

    def __init__(self, bases, coefficients):
        bases = tuple(bases)
        shape = tuple(b.size for b in bases)
        if _is_tensor(coefficients):
            dev = _lib.to_device(coefficients)
            cshape = tuple(dev.shape)
            host = None
        else:
            host = np.array(coefficients, dtype=float, order="C", copy=True)
            cshape = host.shape
            dev = None
        if len(cshape) != len(shape) + 1 or cshape[:-1] != shape:
            raise ValueError(f"stack shape {cshape} does not match member layout {shape} + (count,)")
        if cshape[-1] < 1:
            raise ValueError("stack must hold at least one member")
        _set(self, "bases", bases)
        _set(self, "_host", _freeze(host) if host is not None else None)
        _set(self, "_dev", dev)

    @property
    def count(self) -> int:
        if self._host is not None:
            return self._host.shape[-1]
        return int(self._dev.shape[-1])

    @property
    def coefficients(self) -> np.ndarray:
        if self._host is None:
            _set(self, "_host", _freeze(_lib.to_host(self._dev)))
        return self._host

    @property
    def device_coefficients(self):
        if self._dev is None:
            _set(self, "_dev", _lib.to_device(self._host))
        return self._dev

    def member(self, j: int) -> CoefTensor:
        return CoefTensor(self.bases, np.ascontiguousarray(self.coefficients[..., j]))

    def __repr__(self):
        return f"TensorStack(bases={self.bases!r}, count={self.count})"


@dataclass(frozen=True)
class GatherIndex:
    """Flat-index selection of the member-j / point-j diagonal (S/chebnd.py:84-111)."""

    member_shape: tuple
    count: int
    flat: np.ndarray = field(repr=False)

    def __post_init__(self):
        object.__setattr__(self, "member_shape", tuple(int(d) for d in self.member_shape))
        object.__setattr__(self, "flat", _freeze(np.array(self.flat, dtype=np.int64)))

    def take(self, contracted) -> np.ndarray:
        """Apply the selection to an eval_axis cross product (S/chebnd.py:97-111), on the GPU."""
        rest = self.member_shape[1:]
        expected = rest + (self.count, self.count)
        c = contracted if _is_tensor(contracted) else np.asarray(contracted, dtype=float)
        if tuple(c.shape) != expected:
            raise ValueError(f"expected cross-product shape {expected}, got {tuple(c.shape)}")
        dc = _lib.to_device(c)
        dflat = _lib.to_device_i64(self.flat)
        out_shape = rest + (self.count,)
        out = _lib.empty(out_shape)
        _lib.check(
            _lib.load().cb_gather_take(len(expected), _lib.i64_array(expected), _lib.ptr(dc), int(self.flat.size),
                                       _lib.ptr(dflat), len(out_shape), _lib.i64_array(out_shape), _lib.ptr(out),
                                       _lib.stream_handle()),
            "GatherIndex.take",
        )
        return out if _is_tensor(contracted) else _lib.to_host(out)


# ---------------------------------------------------------------------------------------------
# layout helpers (C ABI pack / unpack)
# ---------------------------------------------------------------------------------------------

def _pack(shape, dense_dev):
    L = _lib.eval_layout(shape)
    out = _lib.empty((L["elems"],))
    _lib.check(_lib.load().cb_pack_eval(len(shape), _lib.i64_array(shape), _lib.ptr(dense_dev), _lib.ptr(out),
                                        _lib.stream_handle()), "pack")
    return out


def _unpack(shape, eval_dev):
    out = _lib.empty(shape)
    _lib.check(_lib.load().cb_unpack_eval(len(shape), _lib.i64_array(shape), _lib.ptr(eval_dev), _lib.ptr(out),
                                          _lib.stream_handle()), "unpack")
    return out


# ---------------------------------------------------------------------------------------------
# basis rows and the private contraction kernels the solver imports (S/solver.py:37-48)
# ---------------------------------------------------------------------------------------------

def _basis_device(points_dev, size: int, clamp: bool, status=None, out=None):
    k = int(points_dev.numel())
    out = _lib.empty((k, size)) if out is None else out
    _lib.check(
        _lib.load().cb_basis_matrix(k, _lib.ptr(points_dev), int(size), _lib.ptr(out), _lib.ptr(status),
                                    1 if clamp else 0, _lib.stream_handle()),
        "basis_matrix",
    )
    return out


def basis_matrix(points, degree: int):
    """B[j, l] = T_l(points[j]), l = 0..degree, by recurrence (S/chebnd.py:114-132)."""
    is_t = _is_tensor(points)
    x = points if is_t else np.asarray(points, dtype=float)
    if x.ndim != 1:
        # the reference clamps first, then rejects the rank
        _host_clamp_check(x)
        raise ValueError("points must be one-dimensional")
    if x.shape[0] == 0:
        raise ValueError("empty point list")
    dx = _lib.to_device(x)
    st = _lib.new_status()
    out = _basis_device(dx, int(degree) + 1, True, st)
    _lib.raise_for_points(st)
    return out if is_t else _lib.to_host(out)


def _host_clamp_check(x):
    if _is_tensor(x):
        x = _lib.to_host(x)
    from .cheb1d import clamp_reference

    clamp_reference(x)


def _row_basis(points, size: int):
    """basis_matrix without validation (S/chebnd.py:135-144)."""
    is_t = _is_tensor(points)
    dx = _lib.to_device(points if is_t else np.asarray(points, dtype=float).ravel())
    out = _basis_device(dx.reshape(-1), int(size), False)
    return out if is_t else _lib.to_host(out)


def _bind_shared(B, member_first):
    """(k, d) x (M, d, rest) -> (M, k, rest) (S/chebnd.py:147-149)."""
    is_t = _is_tensor(member_first)
    dB = _lib.to_device(B)
    dA = _lib.to_device(member_first)
    k, d = dB.shape
    M, d2, rest = dA.shape
    if d != d2:
        raise ValueError("matmul: inner dimensions do not match")
    out = _lib.empty((M, k, rest))
    _lib.check(_lib.load().cb_contract_axis(M, d, rest, 1, k, _lib.ptr(dB), _lib.ptr(dA), _lib.ptr(out), k * rest,
                                            rest, 1, _lib.stream_handle()), "_bind_shared")
    return out if is_t else _lib.to_host(out)


def _bind_rows(B, flat):
    """Row-by-row (k, d) x (d, rest) -> (k, rest) (S/chebnd.py:152-154)."""
    is_t = _is_tensor(flat)
    dB = _lib.to_device(B)
    dF = _lib.to_device(flat)
    k, d = dB.shape
    d2, rest = dF.shape
    if d != d2:
        raise ValueError("matmul: inner dimensions do not match")
    out = _lib.empty((k, rest))
    _lib.check(_lib.load().cb_contract_axis(1, d, rest, 1, k, _lib.ptr(dB), _lib.ptr(dF), _lib.ptr(out), 0, rest, 1,
                                            _lib.stream_handle()), "_bind_rows")
    return out if is_t else _lib.to_host(out)


def _bind_diagonal(B, member_first):
    """Row j of (M, d) against member j of (M, d, rest) -> (M, rest) (S/chebnd.py:157-159)."""
    is_t = _is_tensor(member_first)
    dB = _lib.to_device(B)
    dA = _lib.to_device(member_first)
    M, d = dB.shape
    M2, d2, rest = dA.shape
    if M != M2 or d != d2:
        raise ValueError("matmul: shapes do not match")
    out = _lib.empty((M, rest))
    _lib.check(_lib.load().cb_contract_diagonal(M, d, rest, None, _lib.ptr(dB), 0, _lib.ptr(dA), d * rest, rest, 1,
                                                _lib.ptr(out), rest, 1, None, _lib.stream_handle()), "_bind_diagonal")
    return out if is_t else _lib.to_host(out)


# ---------------------------------------------------------------------------------------------
# build (K1)
# ---------------------------------------------------------------------------------------------

def tensor_coeffs(samples, bases) -> CoefTensor:
    """Coefficient tensor of the interpolant through samples at all node tuples
    (S/chebnd.py:162-190: Algorithm Cnv) — one fused multi-mode GPU build."""
    bases = tuple(bases)
    shape = tuple(b.size for b in bases)
    s_shape = tuple(samples.shape) if _is_tensor(samples) else np.shape(samples)
    if tuple(s_shape) != shape:
        raise ValueError(f"sample shape {tuple(s_shape)} does not match bases {shape}")
    if _is_tensor(samples) and samples.is_cuda:
        ds = samples
        st = _lib.new_status()  # device data: the build's status block reports non-finite samples
    else:
        # host data (numpy / CPU tensor): validated here (S/chebnd.py:181-185), so the build is
        # enqueued without a device status read-back — no host synchronisation in this call
        host = samples.detach().numpy() if _is_tensor(samples) else np.asarray(samples, dtype=float)
        if not np.isfinite(host).all():
            raise ValueError("samples must be finite")
        ds = samples if _is_tensor(samples) else host
        st = None
    ds = _lib.to_device(ds)
    L = _lib.eval_layout(shape)
    out = _lib.empty((L["elems"],))
    _lib.check(_lib.load().cb_tensor_coeffs(len(shape), _lib.i64_array(shape), _lib.ptr(ds), _lib.ptr(out),
                                            _lib.ptr(st), _lib.stream_handle()), "tensor_coeffs")
    if st is not None:
        _lib.raise_for_samples(st)
    return CoefTensor._from_eval_layout(bases, out)


def tensor_coeffs_device(samples_dev, shape, out=None, status=None):
    """Device-resident build without host synchronisation: returns the eval-layout tensor."""
    L = _lib.eval_layout(shape)
    if out is None:
        out = _lib.empty((L["elems"],))
    _lib.check(_lib.load().cb_tensor_coeffs(len(shape), _lib.i64_array(shape), _lib.ptr(samples_dev), _lib.ptr(out),
                                            _lib.ptr(status), _lib.stream_handle()), "tensor_coeffs")
    return out


class BuildEvalGraph:
    """tensor_coeffs + eval_points for fixed shapes and fixed device buffers, captured once as a
    CUDA graph and replayed: the per-sweep refit + evaluate of the solver (S/solver.py:441-449,
    388-397) as ONE submission, for loops whose steps are too small to amortise per-call host work
    (config 1: 65,536 points of a 17 x 17 interpolant).  `samples_dev` (n_1..n_J) and `points_dev`
    (M, J) are read at every replay (update them in place), `out` (M,) is written; no host
    synchronisation and no status checks (validate inputs before, as tensor_coeffs does)."""

    def __init__(self, shape, samples_dev, points_dev, out=None):
        t = _lib.require_cuda()
        self.shape = tuple(int(s) for s in shape)
        self.samples, self.points = samples_dev, points_dev
        self.coef = _lib.empty((_lib.eval_layout(self.shape)["elems"],))
        self.out = out if out is not None else _lib.empty((int(points_dev.shape[0]),))
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(side):
            self._enqueue()  # warm-up outside the capture: smem attributes, tensor-map encoder
        t.cuda.current_stream().wait_stream(side)
        t.cuda.synchronize()
        self.graph = t.cuda.CUDAGraph()
        n0 = int(_lib.load().cb_kernel_launches())
        with t.cuda.graph(self.graph, capture_error_mode="thread_local"):
            self._enqueue()
        self.kernels_per_replay = int(_lib.load().cb_kernel_launches()) - n0  # own kernels in the graph

    def _enqueue(self):
        # one C-ABI call: a single fused launch for small J = 2 tensors, build + evaluation otherwise
        _lib.check(
            _lib.load().cb_build_eval_points(len(self.shape), _lib.i64_array(self.shape), _lib.ptr(self.samples),
                                             int(self.points.shape[0]), _lib.ptr(self.points), _lib.ptr(self.out),
                                             _lib.ptr(self.coef), None, _lib.stream_handle()),
            "build_eval_points",
        )

    def replay(self):
        self.graph.replay()
        return self.out


def stack_coeffs(samples, bases) -> TensorStack:
    """tensor_coeffs for (n_1..n_J, N_P) stacked samples (S/chebnd.py:193-206)."""
    bases = tuple(bases)
    shape = tuple(b.size for b in bases)
    s_shape = tuple(samples.shape) if _is_tensor(samples) else np.shape(samples)
    if len(s_shape) != len(shape) + 1 or tuple(s_shape[:-1]) != shape:
        raise ValueError(f"sample shape {tuple(s_shape)} does not match bases {shape} + (count,)")
    ds = _lib.to_device(samples if _is_tensor(samples) else np.asarray(samples, dtype=float))
    full = tuple(s_shape)
    out = _lib.empty(full)
    st = _lib.new_status()
    if ds.numel() > 0:
        _lib.check(_lib.load().cb_transform_axes(len(full), _lib.i64_array(full), 0, len(shape), _lib.ptr(ds),
                                                 _lib.ptr(out), _lib.ptr(st), 1, _lib.stream_handle()), "stack_coeffs")
    _lib.raise_for_samples(st)
    return TensorStack(bases, out)


# ---------------------------------------------------------------------------------------------
# evaluation (K2, K3)
# ---------------------------------------------------------------------------------------------

def _eval_points_device(shape, coef_dev, points_dev, check: bool = True, dense: bool = False, force_generic=False,
                        out=None):
    """(M, J) reference points -> (M,) values on the device.  coef_dev is the eval layout
    (dense=False) or a dense C-order tensor (dense=True)."""
    if dense:
        coef_dev = _pack(shape, coef_dev)
    M = int(points_dev.shape[0])
    if out is None:
        out = _lib.empty((M,))
    st = _lib.new_status() if check else None
    _lib.check(_lib.load().cb_eval_points(len(shape), _lib.i64_array(shape), _lib.ptr(coef_dev), M,
                                          _lib.ptr(points_dev), _lib.ptr(out), _lib.ptr(st),
                                          1 if force_generic else 0, _lib.stream_handle()), "eval_points")
    if check:
        _lib.raise_for_points(st)
    return out


def eval_points(tensor: CoefTensor, points, check: bool = True):
    """Evaluate one tensor interpolant at M scattered reference points (M, J) -> (M,).

    Additive public form of the solver's batched evaluator (S/solver.py:388-397); equals
    eval_full (S/chebnd.py:315-327) point by point, including clamp_reference semantics."""
    is_t = _is_tensor(points)
    p = points if is_t else np.asarray(points, dtype=float)
    if p.ndim != 2 or p.shape[1] != tensor.ndim:
        raise ValueError(f"expected points of shape (M, {tensor.ndim}), got {tuple(p.shape)}")
    if is_t and not p.is_cuda and p.is_pinned() and p.dtype == _lib.torch().float64 and p.is_contiguous():
        return _eval_points_pinned(tensor, p, check)
    dp = _lib.to_device(p)
    out = _eval_points_device(tensor.shape, tensor.device_coefficients, dp, check=check)
    return _lib.like_input(out, points)


def _eval_points_pinned(tensor: CoefTensor, points, check: bool):
    """Pinned host points -> pinned host values: the C-ABI host pipeline (cb_eval_points_host)
    overlaps the chunked H2D / evaluation / D2H."""
    t = _lib.torch()
    M = int(points.shape[0])
    host_out = t.empty((M,), dtype=t.float64, pin_memory=True)
    if M == 0:
        return host_out
    ws_pts = _lib.empty((M, tensor.ndim))
    ws_out = _lib.empty((M,))
    st = _lib.new_status() if check else None
    _lib.check(_lib.load().cb_eval_points_host(tensor.ndim, _lib.i64_array(tensor.shape),
                                               _lib.ptr(tensor.device_coefficients), M, points.data_ptr(),
                                               host_out.data_ptr(), _lib.ptr(ws_pts), _lib.ptr(ws_out), _lib.ptr(st),
                                               0, _lib.stream_handle()), "eval_points")
    host_st = None
    if check:
        # the status block rides back behind the results: one synchronisation per call
        host_st = t.empty((2,), dtype=t.int64, pin_memory=True)
        host_st.copy_(st, non_blocking=True)
    t.cuda.current_stream().synchronize()
    if check:
        _lib.raise_for_points(host_st)
    return host_out


def eval_full(tensor: CoefTensor, point) -> float:
    """Evaluate one tensor interpolant at a reference point tuple (S/chebnd.py:315-327)."""
    x = np.asarray(point, dtype=float)
    if x.ndim != 1 or x.size != tensor.ndim:
        _host_clamp_check(x)
        raise ValueError(f"expected a {tensor.ndim}-tuple, got shape {x.shape}")
    out = _eval_points_device(tensor.shape, tensor.device_coefficients, _lib.to_device(x.reshape(1, -1)))
    return float(_lib.to_host(out)[0])


def eval_axis(obj, points):
    """Bind the leading variable at a shared list of reference points (S/chebnd.py:209-240).

    (N_2+1, ..., N_J+1, k) for a CoefTensor, (N_2+1, ..., k, N_P) for a TensorStack."""
    is_t = _is_tensor(points)
    x = points if is_t else np.asarray(points, dtype=float)
    if x.ndim != 1 or x.shape[0] == 0:
        if x.ndim != 1 and x.size:
            _host_clamp_check(x)
        raise ValueError("points must be a non-empty one-dimensional list")
    d1 = obj.bases[0].size
    st = _lib.new_status()
    B = _basis_device(_lib.to_device(x), d1, True, st)
    k = int(x.shape[0])
    lib = _lib.load()
    if isinstance(obj, CoefTensor):
        rest = obj.shape[1:]
        R = int(np.prod(rest, dtype=np.int64)) if rest else 1
        A = obj.dense_device()
        out = _lib.empty(rest + (k,))
        _lib.check(lib.cb_contract_axis(1, d1, R, 1, k, _lib.ptr(B), _lib.ptr(A), _lib.ptr(out), 0, 1, k,
                                        _lib.stream_handle()), "eval_axis")
    else:
        A = obj.device_coefficients
        m = obj.count
        rest = tuple(A.shape[1:-1])
        R = int(np.prod(rest, dtype=np.int64)) if rest else 1
        out = _lib.empty(rest + (k, m))
        _lib.check(lib.cb_contract_axis(1, d1, R, m, k, _lib.ptr(B), _lib.ptr(A), _lib.ptr(out), 0, m, k * m,
                                        _lib.stream_handle()), "eval_axis")
    _lib.raise_for_points(st)
    return out if is_t else _lib.to_host(out)


def make_gather_index(member_shape, count: int) -> GatherIndex:
    """Flat-index selection pairing stack member j with point row j (S/chebnd.py:243-272)."""
    member_shape = tuple(int(d) for d in member_shape)
    if len(member_shape) < 1 or any(d < 1 for d in member_shape):
        raise ValueError(f"invalid member shape {member_shape}")
    if count < 1:
        raise ValueError("stack count must be positive")
    rest = int(np.prod(member_shape[1:], dtype=np.int64)) if len(member_shape) > 1 else 1
    total = rest * count * count
    if total > np.iinfo(np.int64).max // 8:
        raise OverflowError("gather index range too large")
    t = _lib.require_cuda()
    flat = t.empty(rest * count, dtype=t.int64, device=_lib.device())
    _lib.check(_lib.load().cb_gather_index(rest, int(count), _lib.ptr(flat), _lib.stream_handle()),
               "make_gather_index")
    return GatherIndex(member_shape=member_shape, count=int(count), flat=_lib.to_host(flat))


def eval_diagonal_batch(stack: TensorStack, points, gather: GatherIndex) -> TensorStack:
    """Bind the leading variable of member j at its own point x_j (S/chebnd.py:275-312)."""
    x = points if _is_tensor(points) else np.asarray(points, dtype=float)
    A = stack.device_coefficients
    member_shape = tuple(A.shape[:-1])
    m = stack.count
    if x.ndim != 1 or x.shape[0] != m:
        raise ValueError(f"need one point per member, got {int(np.prod(x.shape))} points for {m} members")
    if gather.member_shape != member_shape or gather.count != m:
        raise ValueError(
            f"stale gather index: built for {gather.member_shape} x {gather.count}, stack is {member_shape} x {m}"
        )
    d1 = member_shape[0]
    rest = member_shape[1:]
    R = int(np.prod(rest, dtype=np.int64)) if rest else 1
    dx = _lib.to_device(x)
    out = _lib.empty(rest + (m,))
    st = _lib.new_status()
    # stack layout (d1, rest, m): sM = 1, sL = R*m, sR = m ; out (rest, m): oM = 1, oR = m
    _lib.check(_lib.load().cb_contract_diagonal(m, d1, R, _lib.ptr(dx), None, 1, _lib.ptr(A), 1, R * m, m,
                                                _lib.ptr(out), 1, m, _lib.ptr(st), _lib.stream_handle()),
               "eval_diagonal_batch")
    _lib.raise_for_points(st)
    return TensorStack(tuple(stack.bases[1:]), out)


def _eval_grid_device(shape, coef_dev, targets_dev, status=None, work=None, out=None):
    """Device-resident structured evaluation without host synchronisation (K3): eval-layout
    coefficients + per-dim CUDA target vectors -> CUDA (k_1, ..., k_J)."""
    J = len(shape)
    ks = [int(tv.shape[0]) for tv in targets_dev]
    # one C call: the J evaluation matrices (one launch, into one allocation) + the mode passes
    Eall = _lib.empty((sum(k * n for k, n in zip(ks, shape)),))
    lib = _lib.load()
    work_elems = int(lib.cb_eval_grid_workspace(J, _lib.i64_array(shape), _lib.i64_array(ks)))
    if work is None or work.numel() < max(1, work_elems):
        work = _lib.empty((max(1, work_elems),))
    if out is None:
        out = _lib.empty(tuple(ks))
    tv = [tv if tv.dtype == _lib.torch().float64 and tv.is_contiguous() else _lib.to_device(tv) for tv in targets_dev]
    tptrs = (ctypes.c_void_p * J)(*[_lib.ptr(t) for t in tv])
    _lib.check(lib.cb_eval_grid_targets(J, _lib.i64_array(shape), _lib.ptr(coef_dev), _lib.i64_array(ks), tptrs,
                                        _lib.ptr(Eall), _lib.ptr(status), _lib.ptr(out), _lib.ptr(work), work_elems,
                                        _lib.stream_handle()), "eval_grid")
    return out


def eval_grid(tensor: CoefTensor, targets):
    """Structured evaluation on a tensor-product target grid: J successive eval_axis mode products
    (S/chebnd.py:209-233; the paper's pagemtimes evaluation P:385-417).  targets[j] are reference
    coordinates along dim j; the result has shape (k_1, ..., k_J)."""
    J = tensor.ndim
    if len(targets) != J:
        raise ValueError(f"need {J} target lists, got {len(targets)}")
    tvs = []
    for t in targets:
        tv = t if _is_tensor(t) else np.asarray(t, dtype=float)
        if tv.ndim != 1 or tv.shape[0] == 0:
            raise ValueError("points must be a non-empty one-dimensional list")
        tvs.append(_lib.to_device(tv))
    st = _lib.new_status()
    out = _eval_grid_device(tensor.shape, tensor.device_coefficients, tvs, status=st)
    _lib.raise_for_points(st)
    return out if any(_is_tensor(t) for t in targets) else _lib.to_host(out)


# keep the basis type importable from here as in the reference module namespace
ChebBasis1D = ChebBasis1D
