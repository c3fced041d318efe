"""Multi-GPU sharding logic on CPU (gloo, world size 2 / 3) -- no GPU needed.

FAST / EXACT: the sharded all-pairs force (paper_1703_02484_b200/distributed.py)
splits the receiver slots into contiguous per-rank blocks and all-gathers
(fx, fy, flag) records into one (n, 3) buffer.  Here each rank fills its block
with the CPU oracle's forces for its receivers (standing in for the CUDA slot
kernel) and the gather runs over gloo; every rank must end with the full,
bit-identical force array.

FAST-SYM (the default): each rank evaluates the unordered block pairs and
diagonal blocks the library's own split assigns it (bd_sym_shard, the same
function the CUDA launch uses) -- restated here in numpy on the slot order --
and the partials P_r = A_r - B_r are all-reduced over gloo; F = mu P on every
rank must equal the exact oracle to rounding (every unordered pair counted
exactly once), and be identical on all ranks.  tests/test_multirank_gpu.py
runs the same with the CUDA partial kernel on a B200."""

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


def rank_distances(plan):
    D, per = plan["D"], plan["per"]
    out = []
    for k in range(plan["nch"]):
        c = plan["c0"] + k * plan["cs"]
        out.extend(range(1 + c * per, min(1 + (c + 1) * per, D + 1)))
    return out


def sym_partial_np(pos, alpha, L, plan):
    """Numpy restatement of one rank's FAST-SYM partial P_r (slots = particle
    order): diagonal blocks [i0, i1) as directed pairs (receiver side only),
    block pairs (I, I + d mod Mb) for d in the rank's chunks (chunk c holds
    d in [1 + c per, 1 + (c + 1) per), capped at D), both sides (for even Mb,
    d = D only for I < Mb / 2).  Exact reference min image (core.py:81-90)."""
    n = pos.shape[0]
    B, Mb, D = plan["block"], plan["blocks"], plan["D"]
    P = np.zeros((n, 2))

    def blk(I):
        return slice(I * B, min(n, (I + 1) * B))

    def wd(ri, rk):
        d = ri[:, None, :] - rk[None, :, :]
        d = d - np.floor(d / L + 0.5) * L
        r2 = (d * d).sum(-1)
        with np.errstate(divide="ignore", invalid="ignore"):
            w = 1.0 / (r2 * np.sqrt(r2))
        return w[..., None] * d

    for I in range(plan["i0"], plan["i1"]):
        s = blk(I)
        t = wd(pos[s], pos[s])
        idx = np.arange(t.shape[0])
        t[idx, idx] = 0.0
        P[s] += (alpha[s][None, :, None] * t).sum(1)
    even = Mb % 2 == 0
    for d in rank_distances(plan):
        for I in range(Mb):
            if even and d == D and I >= Mb // 2:
                continue
            J = (I + d) % Mb
            si, sj = blk(I), blk(J)
            t = wd(pos[si], pos[sj])
            P[si] += (alpha[sj][None, :, None] * t).sum(1)
            P[sj] -= (alpha[si][:, None, None] * t).sum(0)
    return P


def _sym_worker(rank, world, port, n, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1703_02484_b200.distributed import ShardedLongRange, sym_shard
        rng = np.random.default_rng(5)
        L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
        pos = rng.uniform(0, L, size=(n, 2))
        alpha = np.where(rng.random(n) < 0.5, 3.0, -3.0)
        mu = np.where(alpha > 0, 3.0, -1.5)
        plan = sym_shard(n, rank, world)
        part = torch.from_numpy(sym_partial_np(pos, alpha, L, plan))
        ShardedLongRange(rank, world).reduce(part)  # the product's all-reduce path (gloo here, NCCL on GPUs)
        F = mu[:, None] * part.numpy()
        ref, _ = O.long_range(pos, alpha, mu, L)
        rel = float((np.linalg.norm(F - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())
        gathered = [torch.empty_like(part) for _ in range(world)]
        dist.all_gather(gathered, part)
        same = all(torch.equal(gathered[0], g) for g in gathered)
        out_q.put((rank, rel, bool(same), plan))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(2048, 2), (2500, 3), (1800, 2)])
def test_gloo_fast_sym_partials_allreduce_equal_full(n, world):
    """Every unordered pair once across the ranks (odd / even block counts,
    partial last block), summed by the all-reduce: F = mu P equals the exact
    oracle to rounding on every rank, bit-identical across ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sym_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, rel, same, plan in res:
        assert rel <= 1e-12, (rank, rel, plan)
        assert same, rank
    # the ranks' distances and diagonal ranges tile [1, D] and [0, Mb)
    plans = [r[3] for r in sorted(res, key=lambda r: r[0])]  # by rank
    ds = sorted(d for p in plans for d in rank_distances(p))
    assert ds == list(range(1, plans[0]["D"] + 1))
    assert plans[0]["i0"] == 0 and plans[-1]["i1"] == plans[0]["blocks"]
    assert all(a["i1"] == b["i0"] for a, b in zip(plans, plans[1:]))


@pytest.mark.parametrize("n,world", [(131072, 8), (131072, 2), (1048576, 8), (262144, 4), (65536, 8)])
def test_sym_shard_balance(n, world):
    """Each rank gets the same share of the block pairs (+- one chunk) and of
    the diagonal blocks: the slowest of 8 ranks does <= 1.05x the ideal."""
    from paper_1703_02484_b200.distributed import sym_shard
    plans = [sym_shard(n, r, world) for r in range(world)]
    Mb, D = plans[0]["blocks"], plans[0]["D"]
    work = []
    for p in plans:
        pairs = sum(Mb // 2 if (Mb % 2 == 0 and d == D) else Mb for d in rank_distances(p))
        work.append(pairs + 0.5 * (p["i1"] - p["i0"]))
    total = sum(work)
    assert abs(total - (Mb * D - (Mb // 2 if Mb % 2 == 0 else 0) + 0.5 * Mb)) < 1e-9
    assert max(work) <= 1.05 * total / world + 1.0, work
