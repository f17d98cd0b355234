"""Multi-GPU partitioning of the hot path (one process per GPU, torch.distributed plumbing).

The reference splits node work into contiguous blocks N_b * N_f = N_P on a thread pool
(BlockPlan / partition S/solver.py:61-87, _run_sweep :412-438) with disjoint writes and a barrier
before the refit.  Here the blocks are GPU ranks:

* scattered evaluation (configs 1/2/4): contiguous point shards, coefficients replicated (each
  rank builds them from the same node values — cheaper than any exchange); no data-path
  collective;
* time loop (configs 3/5b): rank r owns node slab [r*S, min(N, (r+1)*S)), S = ceil(N/G).
  - PeerShardedAdvectLoop (the product): the evaluation kernel stores every result of its slab
    straight into all ranks' node-value buffers over NVLink (cb_eval_advected_peers; buffers
    mapped with CUDA IPC), i.e. the all-gather is fused into the compute kernel; node values are
    double-buffered (step t reads buffer t%2, writes (t+1)%2 everywhere) and one stream-ordered
    barrier per step (a 1-element NCCL all-reduce) orders the peers' stores before the next build.
  - ShardedAdvectLoop (baseline): the slab goes to its slot of a padded (G*S) buffer and one NCCL
    all-gather re-assembles the node values.  17^4 and 13^6 are not divisible by 2/4/8, hence the
    padding, unlike the reference's exact-divisor partition.

Per-node arithmetic never depends on the shard, so results are bitwise identical for every
world size (the reference's plan-invariance contract, T/test_solver.py:266-273).
"""

from __future__ import annotations

import math


def shard_range(total: int, rank: int, world: int) -> tuple[int, int, int]:
    """(begin, end, slot) of `rank`'s contiguous shard of `total` items; slot = ceil(total/world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    slot = math.ceil(total / world) if total else 0
    begin = min(total, rank * slot)
    end = min(total, begin + slot)
    return begin, end, slot


class ShardedAdvectLoop:
    """Node-sharded time loop: per step  build (replicated) -> evaluate own slab -> all-gather.

    `backend` supplies build / eval_slab / buffers (CudaStepBackend in the product; the CPU tests
    inject a host backend to exercise the partition and exchange logic under gloo)."""

    def __init__(self, shape, backend, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.shape = tuple(shape)
        self.N = 1
        for s in self.shape:
            self.N *= int(s)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.begin, self.end, self.slot = shard_range(self.N, self.rank, self.world)
        self.backend = backend
        self.full = backend.zeros(self.slot * self.world)

    def run(self, values, steps: int):
        b = self.backend
        self.full[: self.N].copy_(b.to_buffer(values))
        for _ in range(int(steps)):
            b.build(self.full[: self.N])
            mine = self.full[self.rank * self.slot : (self.rank + 1) * self.slot]
            local = b.zeros(self.slot)
            b.eval_slab(self.begin, self.end - self.begin, local)
            if self.world > 1:
                self.dist.all_gather_into_tensor(self.full, local, group=self.group)
            else:
                mine.copy_(local)
        return b.finish(self.full[: self.N].reshape(self.shape))


class PeerShardedAdvectLoop:
    """Node-sharded time loop with the exchange fused into the evaluation (no all-gather):

        step t:  build(V[t%2]) (replicated) -> evaluate own slab, storing each value into every
                 rank's V[(t+1)%2] (NVLink peer stores) -> barrier

    Buffer t%2 is only read by builds of step t and only written by evaluations of step t-1, and
    the barrier of step t-1 separates the two on every rank, so no store races a read (RAW and
    WAR across ranks).  `backend` supplies build / eval_slab_peers / exchange_buffers / barrier
    (CudaStepBackend on GPUs; the CPU tests inject a shared-memory host backend under gloo)."""

    def __init__(self, shape, backend, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.shape = tuple(shape)
        self.N = 1
        for s in self.shape:
            self.N *= int(s)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.begin, self.end, _ = shard_range(self.N, self.rank, self.world)
        self.backend = backend
        self.bufs = [backend.zeros(self.N), backend.zeros(self.N)]
        # dests[b][r]: rank r's buffer b as addressed from this process
        self.dests = backend.exchange_buffers(self.bufs, group)

    def run(self, values, steps: int):
        b = self.backend
        # every rank starts from the same V_0 in its own buffer 0; nobody writes buffer 0 before
        # the barrier that ends step 0
        self.bufs[0].copy_(b.to_buffer(values))
        cur = 0
        for _ in range(int(steps)):
            b.build(self.bufs[cur])
            b.eval_slab_peers(self.begin, self.end - self.begin, self.dests[cur ^ 1])
            b.barrier(self.group)
            cur ^= 1
        out = b.finish(self.bufs[cur].reshape(self.shape).clone())
        if cur != 0:
            # peers' step 0 of a later run() stores into buffer 1: not before this copy is taken
            b.barrier(self.group)
        return out

    def close(self):
        self.backend.close_buffers()
