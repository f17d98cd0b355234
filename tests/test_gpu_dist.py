"""GPU: the fused exchange of the node-sharded loop (cb_eval_advected_peers, CUDA IPC mappings,
dist.PeerShardedAdvectLoop).

* one process, G destination buffers: every destination receives exactly the slab that
  cb_eval_advected computes (bitwise), nothing outside it;
* world size 1 through PeerShardedAdvectLoop == the device-resident loop (bitwise);
* two processes sharing cuda:0 over gloo (IPC-mapped peer buffers, host barrier between steps;
  no kernel waits on another process) == the single-process loop (bitwise), for both step
  parities and a second run on the same mappings.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch

import paper_2307_04688_b200 as cn
from paper_2307_04688_b200 import _lib
from paper_2307_04688_b200.chebnd import tensor_coeffs_device

pytestmark = pytest.mark.gpu


def _bases(shape):
    return [cn.make_basis(n - 1, 0.0, 1.0) for n in shape]


@pytest.mark.parametrize("shape", [(17, 17, 17, 17), (33, 33, 33), (5, 4, 3), (9, 9, 9, 9)])
def test_eval_advected_peers_matches_slab(cuda, shape):
    rng = np.random.default_rng(3)
    J = len(shape)
    A = rng.uniform(-0.5, 0.5, (J, J))
    N = int(np.prod(shape))
    V = _lib.to_device(rng.standard_normal(shape))
    coef = tensor_coeffs_device(V, shape)
    lib = _lib.load()
    sizes = _lib.i64_array(shape)
    lo, hi = _lib.dbl_array([0.0] * J), _lib.dbl_array([1.0] * J)
    ref = _lib.empty((N,))
    lib.cb_eval_advected(J, sizes, _lib.ptr(coef), 0, N, _lib.dbl_array(A), 0.01, lo, hi, 1, _lib.ptr(ref),
                         _lib.stream_handle())
    begin, end = N // 3, N // 3 + (N + 1) // 2
    dests = [torch.zeros(N, dtype=torch.float64, device=cuda) for _ in range(3)]
    arr = (ctypes.c_void_p * 3)(*[_lib.ptr(d) for d in dests])
    _lib.check(lib.cb_eval_advected_peers(J, sizes, _lib.ptr(coef), begin, end - begin, _lib.dbl_array(A), 0.01, lo,
                                          hi, 1, arr, 3, _lib.stream_handle()), "peers")
    r = _lib.to_host(ref)
    for d in dests:
        h = _lib.to_host(d)
        assert np.array_equal(h[begin:end], r[begin:end])
        assert not h[:begin].any() and not h[end:].any()


def test_eval_advected_peers_rejects_bad_args(cuda):
    lib = _lib.load()
    shape = (5, 5)
    coef = tensor_coeffs_device(_lib.to_device(np.ones(shape)), shape)
    arr = (ctypes.c_void_p * 1)(None)
    with pytest.raises(ValueError):
        _lib.check(lib.cb_eval_advected_peers(2, _lib.i64_array(shape), _lib.ptr(coef), 0, 25,
                                              _lib.dbl_array(np.zeros((2, 2))), 0.01, _lib.dbl_array([0, 0]),
                                              _lib.dbl_array([1, 1]), 1, arr, 1, _lib.stream_handle()))
    with pytest.raises(ValueError):
        _lib.check(lib.cb_eval_advected_peers(2, _lib.i64_array(shape), _lib.ptr(coef), 0, 25,
                                              _lib.dbl_array(np.zeros((2, 2))), 0.01, _lib.dbl_array([0, 0]),
                                              _lib.dbl_array([1, 1]), 1, arr, 9, _lib.stream_handle()))


@pytest.mark.parametrize("shape,steps", [((9, 9, 9), 3), ((17, 17, 17, 17), 4)])
def test_peer_loop_world1(cuda, shape, steps):
    from paper_2307_04688_b200.dist import PeerShardedAdvectLoop
    from paper_2307_04688_b200.loop import CudaStepBackend

    rng = np.random.default_rng(5)
    J = len(shape)
    A = rng.uniform(-0.5, 0.5, (J, J))
    V0 = rng.standard_normal(shape)
    loop = PeerShardedAdvectLoop(shape, CudaStepBackend(_bases(shape), A, 0.01))
    got = _lib.to_host(loop.run(V0, steps))
    ref = cn.advect_loop(V0, _bases(shape), A, 0.01, steps)
    assert np.array_equal(got, ref)
    loop.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, A, V0, steps, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_04688_b200.dist import PeerShardedAdvectLoop
        from paper_2307_04688_b200.loop import CudaStepBackend

        loop = PeerShardedAdvectLoop(shape, CudaStepBackend(_bases(shape), A, 0.01))
        v1 = _lib.to_host(loop.run(V0, steps))
        v2 = _lib.to_host(loop.run(V0, steps + 1))
        dist.barrier()
        loop.close()
        q.put((rank, v1, v2, None))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(9, 9, 9), (17, 17, 17, 17)])
def test_peer_loop_two_processes_one_gpu(cuda, shape):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(9)
    J = len(shape)
    A = rng.uniform(-0.5, 0.5, (J, J))
    V0 = rng.standard_normal(shape)
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, A, V0, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, v1, v2, err = q.get(timeout=300)
        assert err is None, err
        res[r] = (v1, v2)
    for p in procs:
        p.join(timeout=60)
    ref1 = cn.advect_loop(V0, _bases(shape), A, 0.01, steps)
    ref2 = cn.advect_loop(V0, _bases(shape), A, 0.01, steps + 1)
    for r in range(2):
        assert np.array_equal(res[r][0], ref1), (r, np.abs(res[r][0] - ref1).max())
        assert np.array_equal(res[r][1], ref2), (r, np.abs(res[r][1] - ref2).max())
