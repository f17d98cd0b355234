"""CPU, world_size 2 over gloo: the node-sharded time loop (paper_2307_04688_b200/dist.py) —
contiguous padded slabs, one all-gather per step — reproduces the single-process loop bitwise.

The GPU kernels cannot run here, so the test injects a host step backend built from the oracle
(test infrastructure); the partition / exchange / reassembly logic under test is the product's.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_04688_b200.dist import ShardedAdvectLoop, shard_range


class HostBackend:
    """Oracle-backed stand-in for CudaStepBackend (same interface)."""

    def __init__(self, shape, A, dt):
        from oracle import cheb_oracle as orc

        self.orc = orc
        self.shape = tuple(shape)
        self.T, self.S = orc.advect_points(self.shape, A, dt)
        self.C = None

    def zeros(self, n):
        return torch.zeros(int(n), dtype=torch.float64)

    def to_buffer(self, values):
        return torch.as_tensor(np.ascontiguousarray(values, dtype=float)).reshape(-1)

    def build(self, full_values):
        self.C = self.orc.tensor_coeffs(full_values.numpy().reshape(self.shape))

    def eval_slab(self, begin, count, out_view):
        if count <= 0:
            return
        v = self.orc.eval_points(self.C, self.T[begin:begin + count]) - self.S[begin:begin + count]
        out_view[:count].copy_(torch.from_numpy(v))

    def finish(self, full_values):
        return full_values


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, A, V0, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        loop = ShardedAdvectLoop(shape, HostBackend(shape, A, 0.01))
        V = loop.run(V0, steps)
        q.put((rank, V.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(5, 5, 5), (4, 3, 5)])
def test_sharded_loop_world2_matches_single(shape):
    from oracle import cheb_oracle as orc

    rng = np.random.default_rng(7)
    J = len(shape)
    A = rng.uniform(-0.5, 0.5, (J, J))
    V0 = rng.standard_normal(shape)
    ref = orc.advect_loop(V0, A, 0.01, 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, A, V0, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert np.array_equal(res[r], ref), (r, np.abs(res[r] - ref).max())


def test_shard_range_covers_exactly():
    for total in (0, 1, 7, 83521, 4826809):
        for world in (1, 2, 3, 4, 8):
            pieces = [shard_range(total, r, world) for r in range(world)]
            slot = pieces[0][2]
            assert all(p[2] == slot for p in pieces)
            covered = []
            for b, e, _ in pieces:
                assert 0 <= b <= e <= total and e - b <= slot
                covered.extend(range(b, e)) if total < 100 else None
            if total < 100:
                assert covered == list(range(total))
            assert sum(e - b for b, e, _ in pieces) == total
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


# ------------------------------------------------------------------------------------------------
# Fused exchange (PeerShardedAdvectLoop): every rank stores its slab into all ranks' buffers.
# Here the "peer memory" is shared CPU tensors (torch shared memory) standing in for CUDA IPC
# mappings; the ping-pong / barrier protocol under test is the product's.
# ------------------------------------------------------------------------------------------------

class SharedPeerBackend(HostBackend):
    def __init__(self, shape, A, dt, shared, rank):
        super().__init__(shape, A, dt)
        self.shared = shared    # shared[r][b]: rank r's buffer b (shared memory)
        self.rank = rank
        self.nz = 0

    def zeros(self, n):
        t = self.shared[self.rank][self.nz]
        self.nz += 1
        t.zero_()
        return t

    def exchange_buffers(self, bufs, group=None):
        world = len(self.shared)
        return [[self.shared[r][b] for r in range(world)] for b in range(len(bufs))]

    def eval_slab_peers(self, begin, count, dests):
        if count <= 0:
            return
        v = torch.from_numpy(self.orc.eval_points(self.C, self.T[begin:begin + count]) - self.S[begin:begin + count])
        for d in dests:
            d[begin:begin + count].copy_(v)

    def barrier(self, group=None):
        dist.barrier(group=group)

    def close_buffers(self):
        pass


def _peer_worker(rank, world, port, shape, A, V0, steps, shared, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_04688_b200.dist import PeerShardedAdvectLoop

        loop = PeerShardedAdvectLoop(shape, SharedPeerBackend(shape, A, 0.01, shared, rank))
        V1 = loop.run(V0, steps)
        V2 = loop.run(V0, steps + 1)   # a second run on the same buffers (other parity)
        q.put((rank, V1.numpy().copy(), V2.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,world", [((5, 5, 5), 2), ((4, 3, 5), 3)])
def test_peer_loop_matches_single(shape, world):
    from oracle import cheb_oracle as orc

    rng = np.random.default_rng(11)
    J = len(shape)
    A = rng.uniform(-0.5, 0.5, (J, J))
    V0 = rng.standard_normal(shape)
    N = int(np.prod(shape))
    shared = [[torch.zeros(N, dtype=torch.float64).share_memory_() for _ in range(2)] for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, shape, A, V0, 3, shared, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, v1, v2 = q.get(timeout=120)
        res[r] = (v1, v2)
    for p in procs:
        p.join(timeout=60)
    ref1 = orc.advect_loop(V0, A, 0.01, 3)
    ref2 = orc.advect_loop(V0, A, 0.01, 4)
    for r in range(world):
        assert np.array_equal(res[r][0], ref1), (r, np.abs(res[r][0] - ref1).max())
        assert np.array_equal(res[r][1], ref2), (r, np.abs(res[r][1] - ref2).max())


def test_cuda_backend_barrier_takes_nccl_branch(monkeypatch):
    """CudaStepBackend.barrier under an nccl group (world > 1) is the stream-ordered 1-element NCCL
    all-reduce on the compute stream (no host synchronize, no host barrier); under gloo it is the
    device synchronize + host barrier.  Host logic only: torch.distributed is stubbed."""
    from paper_2307_04688_b200 import _lib
    from paper_2307_04688_b200.loop import CudaStepBackend

    calls = []
    monkeypatch.setattr(_lib, "require_cuda", lambda: torch)
    be = object.__new__(CudaStepBackend)  # no device buffers needed for the branch logic
    be._flag = object()
    monkeypatch.setattr(dist, "is_initialized", lambda: True)
    monkeypatch.setattr(dist, "get_world_size", lambda group=None: 2)
    monkeypatch.setattr(dist, "all_reduce", lambda t, group=None: calls.append(("all_reduce", t)))
    monkeypatch.setattr(dist, "barrier", lambda group=None: calls.append(("barrier", None)))
    monkeypatch.setattr(torch.cuda, "synchronize", lambda *a, **k: calls.append(("synchronize", None)))
    monkeypatch.setattr(dist, "get_backend", lambda group=None: "nccl")
    be.barrier()
    assert calls == [("all_reduce", be._flag)]
    calls.clear()
    monkeypatch.setattr(dist, "get_backend", lambda group=None: "gloo")
    be.barrier()
    assert [c[0] for c in calls] == ["synchronize", "barrier"]
    calls.clear()
    monkeypatch.setattr(dist, "get_world_size", lambda group=None: 1)
    be.barrier()
    assert calls == []
