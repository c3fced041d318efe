"""Multi-GPU sharding of the all-pairs force (one process per GPU).

Only the O(N^2) force is partitioned; every rank holds the
full simulation state.  The O(N) path -- integrate, triangulation
maintenance, Verlet lists, overlap correction -- runs as identical,
deterministic replicas on every rank, so no further collective is needed
(its per-pass global barriers would cost more over NVLink than the work;
DESIGN.md §7).  Two decompositions:

  * FAST / EXACT (`force`): each rank computes the forces of its own
    contiguous block of receiver slots and the (fx, fy, flag) records of all
    slots are all-gathered (24 B x N per step).  Each receiver's sum is
    computed whole by one rank in one order, so the forces are
    bit-identical for every world size.
  * FAST-SYM (`force_sym`, the default precision): each rank evaluates its
    share of the unordered block pairs and writes an (n, 2) partial; the
    partials are summed by an all-reduce (16 B x N).  The result is
    identical on every rank of one run, but its last bits depend on the
    world size and on the all-reduce's summation order (NCCL picks ring or
    tree); against the single-GPU FAST-SYM forces it agrees to ~1e-15
    relative (tests/test_distributed.py, tests/test_multirank_gpu.py).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

from ._abi import BD_LR_FAST_SYM
from ._lib import check, lib


@dataclass
class Shard:
    rank: int
    world: int
    chunk: int  # slots per rank (last rank may own fewer)

    def bounds(self, n: int):
        s0 = min(n, self.rank * self.chunk)
        return s0, min(n, s0 + self.chunk)


# receiver slots per rank are a multiple of this: every rank's receiver
# blocks then coincide with the single-GPU blocks (FS_RPB = 128 slots per CTA
# in csrc/bd_allpairs_fast.cuh), so per-block decisions (the generic
# image path) and hence the bits are the same for every world size
SLOT_ALIGN = 256


def shard_for(n: int, rank: int, world: int) -> Shard:
    chunk = (n + world - 1) // world
    return Shard(rank, world, (chunk + SLOT_ALIGN - 1) // SLOT_ALIGN * SLOT_ALIGN)


def sym_shard(n: int, rank: int, world: int) -> dict:
    """The FAST-SYM work split of one rank (bd_sym_shard; host-only, no GPU
    needed): which unordered block pairs and diagonal blocks it evaluates."""
    out = (ctypes.c_int64 * 11)()
    check(lib().bd_sym_shard(int(n), int(rank), int(world), out), "bd_sym_shard")
    keys = ("block", "blocks", "D", "chunks", "per", "c0", "cs", "nch", "reserved", "i0", "i1")
    return dict(zip(keys, (int(v) for v in out)))


class ShardedLongRange:
    """Receiver-slot sharding of the all-pairs force over a process group.

    `gather(buf, mine)` must all-gather `mine` (a view of `buf` at this rank's
    offset) into `buf`; by default torch.distributed.all_gather_into_tensor on
    the given group (NCCL on GPUs)."""

    def __init__(self, rank: int, world: int, group=None, gather=None, reduce=None):
        self.rank = int(rank)
        self.world = int(world)
        self.group = group
        self._gather = gather
        self._reduce = reduce
        self._buf = None
        self._part = None

    @classmethod
    def from_env(cls, group=None):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_rank(group), dist.get_world_size(group), group)
        return cls(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), group)

    def gather(self, buf, mine):
        if self._gather is not None:
            return self._gather(buf, mine)
        import torch.distributed as dist
        dist.all_gather_into_tensor(buf, mine, group=self.group)

    def buffer(self, n: int, device):
        import torch
        sh = shard_for(n, self.rank, self.world)
        rows = sh.chunk * self.world
        if self._buf is None or self._buf.shape[0] != rows or self._buf.device != device:
            self._buf = torch.zeros((rows, 3), dtype=torch.float64, device=device)
        return self._buf, sh

    def reduce(self, part):
        """Sum the per-rank FAST-SYM partials in place (all-reduce)."""
        if self._reduce is not None:
            return self._reduce(part)
        import torch.distributed as dist
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group)

    def part_buffer(self, n: int, device):
        import torch
        if self._part is None or self._part.shape[0] != n or self._part.device != device:
            self._part = torch.zeros((n, 2), dtype=torch.float64, device=device)
        return self._part

    def force_sym(self, state, params, stream):
        """FAST-SYM for a sharded group: this rank's share of the block pairs
        -> per-slot partial, all-reduce (NCCL), finish."""
        n = int(params.n)
        part = self.part_buffer(n, self._device_of(state))
        L = lib()
        check(L.bd_force_sym_partial(ctypes.byref(state), ctypes.byref(params), self.rank, self.world,
                                     ctypes.c_void_p(part.data_ptr()), stream), "bd_force_sym_partial")
        self.reduce(part)
        check(L.bd_force_sym_finish(ctypes.byref(state), ctypes.byref(params), ctypes.c_void_p(part.data_ptr()),
                                    stream), "bd_force_sym_finish")

    def force(self, state, params, stream):
        """bd_force for a sharded group: prepare, own slots, all-gather, finish."""
        if int(params.lr_precision) == BD_LR_FAST_SYM:
            return self.force_sym(state, params, stream)
        n = int(params.n)
        buf, sh = self.buffer(n, self._device_of(state))
        s0, s1 = sh.bounds(n)
        L = lib()
        check(L.bd_force_prepare(ctypes.byref(state), ctypes.byref(params), stream), "bd_force_prepare")
        check(L.bd_force_slots(ctypes.byref(state), ctypes.byref(params), s0, s1, ctypes.c_void_p(buf.data_ptr()),
                               stream), "bd_force_slots")
        mine = buf[self.rank * sh.chunk:(self.rank + 1) * sh.chunk]
        self.gather(buf, mine)
        check(L.bd_force_finish(ctypes.byref(state), ctypes.byref(params), ctypes.c_void_p(buf.data_ptr()), stream),
              "bd_force_finish")

    def _device_of(self, state):
        import torch
        return torch.device("cuda", torch.cuda.current_device())


class SequentialShards(ShardedLongRange):
    """All `world` shards computed one after another on this GPU (the
    single-GPU check of the sharded path: same slices, same buffer layout,
    the all-gather replaced by the identity)."""

    def __init__(self, world: int):
        super().__init__(0, world, gather=lambda buf, mine: None)

    def force(self, state, params, stream):
        n = int(params.n)
        if int(params.lr_precision) == BD_LR_FAST_SYM:
            # every rank's partial in turn, summed in rank order (the all-reduce)
            import torch
            L = lib()
            dev = self._device_of(state)
            total = torch.zeros((n, 2), dtype=torch.float64, device=dev)
            part = torch.zeros((n, 2), dtype=torch.float64, device=dev)
            for r in range(self.world):
                check(L.bd_force_sym_partial(ctypes.byref(state), ctypes.byref(params), r, self.world,
                                             ctypes.c_void_p(part.data_ptr()), stream), "bd_force_sym_partial")
                total += part
            check(L.bd_force_sym_finish(ctypes.byref(state), ctypes.byref(params), ctypes.c_void_p(total.data_ptr()),
                                        stream), "bd_force_sym_finish")
            return
        buf, _ = self.buffer(n, self._device_of(state))
        L = lib()
        check(L.bd_force_prepare(ctypes.byref(state), ctypes.byref(params), stream), "bd_force_prepare")
        for r in range(self.world):
            s0, s1 = shard_for(n, r, self.world).bounds(n)
            check(L.bd_force_slots(ctypes.byref(state), ctypes.byref(params), s0, s1,
                                   ctypes.c_void_p(buf.data_ptr()), stream), "bd_force_slots")
        check(L.bd_force_finish(ctypes.byref(state), ctypes.byref(params), ctypes.c_void_p(buf.data_ptr()), stream),
              "bd_force_finish")
