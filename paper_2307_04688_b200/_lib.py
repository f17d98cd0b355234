"""ctypes binding of libchebnash_b200.so (the C ABI in include/chebnash_b200.h) plus the device
plumbing the shim needs: torch CUDA buffers, the current stream and the status block.

There is no CPU fallback: every numeric call goes through the CUDA library, and calling one on a
host without a CUDA device raises RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CHEBNASH_B200_LIB: load another build of the same library (tools/ experiments only)
LIB_PATH = os.environ.get("CHEBNASH_B200_LIB") or os.path.join(_HERE, "libchebnash_b200.so")

_c_int = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_i64p = ctypes.POINTER(ctypes.c_int64)
_dblp = ctypes.POINTER(ctypes.c_double)

MAX_PLAYERS = 8          # CB_MAX_PLAYERS
MAX_CONTROL_NODES = 32   # CB_MAX_CONTROL_NODES


class CbGame(ctypes.Structure):
    """cb_game_t (include/chebnash_b200.h): GameSpec + derived node tables for the device solver."""

    _fields_ = [
        ("J", ctypes.c_int),
        ("np", ctypes.c_int * MAX_PLAYERS),
        ("nu", ctypes.c_int * MAX_PLAYERS),
        ("h", ctypes.c_double),
        ("delta", ctypes.c_double),
        ("P_max", ctypes.c_double),
        ("U_max", ctypes.c_double),
        ("tol", ctypes.c_double),
        ("A", ctypes.c_double * MAX_PLAYERS),
        ("phi", ctypes.c_double * MAX_PLAYERS),
        ("K", (ctypes.c_double * MAX_PLAYERS) * MAX_PLAYERS),
        ("beta", ctypes.c_double * MAX_PLAYERS),
        ("c", ctypes.c_double * MAX_PLAYERS),
        ("m", ctypes.c_double * MAX_PLAYERS),
        ("unodes", (ctypes.c_double * MAX_CONTROL_NODES) * MAX_PLAYERS),
        ("rnodes", (ctypes.c_double * MAX_CONTROL_NODES) * MAX_PLAYERS),
    ]


_gamep = ctypes.POINTER(CbGame)

# name -> (restype, argtypes); must match include/chebnash_b200.h
SIGNATURES = {
    "cb_abi_version": (_c_int, []),
    "cb_last_error": (ctypes.c_char_p, []),
    "cb_kernel_launches": (_c_i64, []),
    "cb_last_eval_plan": (ctypes.c_char_p, []),
    "cb_runtime_info": (_c_int, [ctypes.POINTER(_c_int)] * 4),
    "cb_eval_layout": (_c_int, [_c_int, _i64p, _i64p]),
    "cb_pack_eval": (_c_int, [_c_int, _i64p, _vp, _vp, _vp]),
    "cb_unpack_eval": (_c_int, [_c_int, _i64p, _vp, _vp, _vp]),
    "cb_tensor_coeffs": (_c_int, [_c_int, _i64p, _vp, _vp, _vp, _vp]),
    "cb_transform_axes": (_c_int, [_c_int, _i64p, _c_int, _c_int, _vp, _vp, _vp, _c_int, _vp]),
    "cb_eval_points": (_c_int, [_c_int, _i64p, _vp, _c_i64, _vp, _vp, _vp, _c_int, _vp]),
    "cb_build_eval_points": (_c_int, [_c_int, _i64p, _vp, _c_i64, _vp, _vp, _vp, _vp, _vp]),
    "cb_eval_points_host": (_c_int, [_c_int, _i64p, _vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _c_int, _vp]),
    "cb_eval_advected": (_c_int, [_c_int, _i64p, _vp, _c_i64, _c_i64, _dblp, _c_dbl, _dblp, _dblp, _c_int, _vp, _vp]),
    "cb_eval_advected_peers": (
        _c_int, [_c_int, _i64p, _vp, _c_i64, _c_i64, _dblp, _c_dbl, _dblp, _dblp, _c_int, ctypes.POINTER(_vp), _c_int, _vp]
    ),
    "cb_ipc_export": (_c_int, [_vp, _vp]),
    "cb_ipc_import": (_c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "cb_ipc_close": (_c_int, [_vp]),
    "cb_advect_loop": (_c_int, [_c_int, _i64p, _vp, _vp, _vp, _c_int, _dblp, _c_dbl, _dblp, _dblp, _vp, _c_int, _vp]),
    "cb_contract_axis": (_c_int, [_c_i64, _c_int, _c_i64, _c_i64, _c_int, _vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _vp]),
    "cb_contract_diagonal": (
        _c_int,
        [_c_i64, _c_int, _c_i64, _vp, _vp, _c_int, _vp, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _vp, _vp],
    ),
    "cb_derivative": (_c_int, [_c_i64, _c_int, _vp, _vp, _vp]),
    "cb_basis_matrix": (_c_int, [_c_i64, _vp, _c_int, _vp, _vp, _c_int, _vp]),
    "cb_gather_index": (_c_int, [_c_i64, _c_i64, _vp, _vp]),
    "cb_gather_take": (_c_int, [_c_int, _i64p, _vp, _c_i64, _vp, _c_int, _i64p, _vp, _vp]),
    "cb_eval_grid_workspace": (_c_i64, [_c_int, _i64p, _i64p]),
    "cb_eval_grid": (_c_int, [_c_int, _i64p, _vp, _i64p, ctypes.POINTER(_vp), _vp, _vp, _c_i64, _vp]),
    "cb_eval_grid_targets": (_c_int, [_c_int, _i64p, _vp, _i64p, ctypes.POINTER(_vp), _vp, _vp, _vp, _vp, _c_i64,
                                      _vp]),
    "cb_solver_drift_elems": (_c_i64, [_gamep]),
    "cb_solver_drift_layout": (_c_int, [_gamep, _vp, _vp, _vp]),
    "cb_bellman_sweep": (_c_int, [_gamep, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "cb_solve_work_bytes": (_c_i64, [_gamep, _c_i64]),
    "cb_solve": (_c_int, [_gamep, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _i64p, ctypes.POINTER(_c_int), _vp]),
    "cb_maximise_rows": (_c_int, [_c_i64, _c_int, _vp, _vp, _vp, _vp, _c_int, _vp]),
    "cb_simulate": (_c_int, [_gamep, _c_i64, _vp, _vp, _c_i64, _vp, _vp, _vp]),
    "cb_lq": (_c_int, [_gamep, _vp, _vp, _c_i64, _c_dbl, _c_int, _i64p, _vp]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load the shared library (raises OSError with a build hint when it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise OSError(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(nvcc, sm_100a).  There is no CPU fallback."
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class CudaLibraryError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().cb_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg or what)
        if rc == 2:
            raise FloatingPointError(msg or what)
        if rc == 3:
            raise RuntimeError(msg or what)
        raise CudaLibraryError(f"{what}: {msg}" if what else msg)


def i64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_int64 * max(1, len(vals)))(*vals)


def dbl_array(values) -> ctypes.Array:
    vals = [float(v) for v in np.asarray(values, dtype=float).ravel()]
    return (ctypes.c_double * max(1, len(vals)))(*vals)


def eval_layout(sizes) -> dict:
    """Host-side eval-layout plan (cb_eval_layout)."""
    lib = load()
    out = (ctypes.c_int64 * 6)()
    check(lib.cb_eval_layout(len(sizes), i64_array(sizes), out), "cb_eval_layout")
    return {"q": out[0], "R": out[1], "R8": out[2], "K": out[3], "Kp": out[4], "elems": out[5]}


# ---------------------------------------------------------------------------------------------
# device plumbing (torch is only the allocator / stream provider)
# ---------------------------------------------------------------------------------------------

def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_2307_04688_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback"
        )
    load()
    return t


def device():
    t = require_cuda()
    return t.device("cuda", t.cuda.current_device())


def stream_handle() -> int:
    t = require_cuda()
    return int(t.cuda.current_stream().cuda_stream)


def to_device(a):
    """fp64 C-contiguous CUDA tensor from array-like or tensor (no copy when already there)."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        if a.is_cuda and a.dtype == t.float64 and a.is_contiguous():
            return a
        pinned = (not a.is_cuda) and a.is_pinned()
        return a.to(device=device(), dtype=t.float64, non_blocking=pinned).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=float))
    if not arr.flags.writeable:  # read-only views (frozen reference-style arrays): torch wants a copy
        arr = arr.copy()
    host = t.from_numpy(arr)
    if arr.nbytes >= (1 << 20):
        host = host.pin_memory()
        return host.to(device(), non_blocking=True)
    return host.to(device())


def to_device_i64(a):
    t = require_cuda()
    if isinstance(a, t.Tensor):
        return a.to(device=device(), dtype=t.int64).contiguous()
    return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64))).to(device())


def empty(shape, dtype=None):
    t = require_cuda()
    return t.empty(tuple(int(s) for s in shape), dtype=dtype or t.float64, device=device())


def to_host(x) -> np.ndarray:
    """Device tensor -> numpy.  Large results go through a pinned buffer from torch's caching host
    allocator (a pageable D2H copy runs at a fraction of PCIe bandwidth)."""
    x = x.detach()
    if not x.is_cuda or x.numel() * x.element_size() < (1 << 20):
        return x.cpu().numpy()
    t = torch()
    host = t.empty(x.shape, dtype=x.dtype, pin_memory=True)
    host.copy_(x, non_blocking=True)
    t.cuda.current_stream().synchronize()
    return host.numpy()


def like_input(out, ref):
    """Return `out` (CUDA) in the kind of `ref`: CUDA tensor -> as is; CPU tensor -> pinned CPU
    tensor (one D2H copy); anything else -> numpy."""
    t = torch()
    if isinstance(ref, t.Tensor):
        if ref.is_cuda:
            return out
        host = t.empty(out.shape, dtype=out.dtype, pin_memory=True)
        host.copy_(out, non_blocking=True)
        t.cuda.current_stream().synchronize()
        return host
    return to_host(out)


def ptr(x) -> int | None:
    return None if x is None else int(x.data_ptr())


def new_status():
    t = require_cuda()
    return t.zeros(2, dtype=t.int64, device=device())


def read_status(st) -> tuple[int, int, float]:
    w = to_host(st)
    nonfinite = int(w[0] & 0xFFFFFFFF)
    domain = int((w[0] >> 32) & 0xFFFFFFFF)
    worst = float(np.array([w[1]], dtype=np.int64).view(np.float64)[0])
    return nonfinite, domain, worst


def raise_for_points(st) -> None:
    """clamp_reference error semantics (S/cheb1d.py:127-135)."""
    nonfinite, domain, worst = read_status(st)
    if nonfinite:
        raise ValueError("evaluation points must be finite")
    if domain:
        raise ValueError(f"evaluation point outside [-1, 1] beyond tolerance: |x| = {worst}")


def raise_for_samples(st, what: str = "samples must be finite") -> None:
    nonfinite, _, _ = read_status(st)
    if nonfinite:
        raise ValueError(what)
