"""Multi-GPU sharding logic on CPU (gloo, world size 2) -- no GPU needed.

The sharded all-pairs force (paper_1703_02484_b200/distributed.py) splits the
receiver slots into contiguous per-rank blocks and all-gathers (fx, fy, flag)
records into one (n, 3) buffer.  Here each rank fills its block with the CPU
oracle's forces for its receivers (standing in for the CUDA slot kernel) and
the gather runs over gloo; every rank must end with the full, bit-identical
force array."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_02484_b200.distributed import ShardedLongRange, shard_for


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,world", [(1000, 2), (1001, 2), (7, 3), (131072, 8)])
def test_shard_bounds_partition(n, world):
    seen = np.zeros(n, dtype=int)
    for r in range(world):
        s0, s1 = shard_for(n, r, world).bounds(n)
        seen[s0:s1] += 1
    assert (seen == 1).all()


def _worker(rank, world, port, n, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes
        from oracle import oracle as O
        rng = np.random.default_rng(3)
        L = 40.0
        pos = rng.uniform(0, L, size=(n, 2))
        alpha = rng.normal(size=n)
        mu = rng.normal(size=n)

        def gloo_gather(buf, mine):
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine.contiguous())
            buf.copy_(torch.cat(parts, 0))

        sh = ShardedLongRange(rank, world, gather=gloo_gather)
        buf, shard = sh.buffer(n, torch.device("cpu"))
        s0, s1 = shard.bounds(n)
        lib = O.lib()
        lib.bdo_long_range_range.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                                                       ctypes.c_int64, ctypes.c_int64,
                                                                       ctypes.c_void_p, ctypes.c_void_p]
        out = np.zeros((n, 2))
        err = np.zeros(n, np.int64)
        lib.bdo_long_range_range(pos.ctypes.data, alpha.ctypes.data, mu.ctypes.data, n, L, 1, s0, s1,
                                 out.ctypes.data, err.ctypes.data)
        mine = buf[rank * shard.chunk:(rank + 1) * shard.chunk]
        k = s1 - s0
        mine[:k, 0:2] = torch.from_numpy(out[s0:s1])
        mine[:k, 2] = torch.from_numpy(err[s0:s1].astype(np.float64))
        sh.gather(buf, mine)
        full, ferr = O.long_range(pos, alpha, mu, L)
        ok = np.array_equal(buf[:n, 0:2].numpy(), full) and np.array_equal(buf[:n, 2].numpy().astype(np.int64), ferr)
        out_q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [500, 501])
def test_gloo_world2_sharded_forces_equal_full(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
