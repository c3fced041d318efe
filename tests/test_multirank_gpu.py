"""The multi-rank path of the default FAST-SYM force on one B200: two ranks
(processes) share cuda:0 and talk over gloo instead of NCCL (only one GPU
per box here; the data path -- bd_force_sym_partial per rank, all-reduce of
the (n, 2) partials, bd_force_sym_finish, the replicated O(N) step -- is the
NCCL one, only the transport differs).

  * the forces of the sharded step equal the single-rank FAST-SYM forces to
    rounding (|dF|/|F| <= 1e-12: every unordered pair once, summed in
    another order);
  * both ranks hold bit-identical positions and triangulations after every
    step (the O(N) path is a deterministic replica);
  * bench.py --gpus 2 (re-launched under torch.distributed.run by itself)
    runs two ranks and reports n_gpus 2.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sim(rec, sharding=None):
    from helpers import product_sim
    sim = product_sim(rec, precision="fast-sym")
    sim.sharding = sharding
    return sim


def _rank(rank, world, port, q):
    import hashlib

    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from golden_io import load
        from paper_1703_02484_b200.distributed import ShardedLongRange
        torch.cuda.set_device(0)

        def reduce(part):
            h = part.cpu()
            dist.all_reduce(h)
            part.copy_(h.to(part.device))

        rec = load("cfg1_lr_c0_n1024")
        sim = _sim(rec, ShardedLongRange(rank, world, reduce=reduce))
        forces, digests = [], []
        for _ in range(3):
            sim.step()
            forces.append(sim.sys.forces_t.cpu().numpy().copy())
            h = hashlib.sha256(sim.sys.positions_t.cpu().numpy().tobytes())
            for v in sim.tri.arrays().values():
                h.update(v.tobytes())
            digests.append(h.hexdigest())
        q.put((rank, forces, digests))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fast_sym_ranks_on_one_gpu(world):
    import torch.multiprocessing as mp
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import load
    rec = load("cfg1_lr_c0_n1024")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    # every rank: the same state after every step
    for r in res[1:]:
        assert r[2] == res[0][2]
    # step 0 forces (same input state) vs the single-rank FAST-SYM
    single = _sim(rec)
    single.step()
    f1 = single.sys.forces_t.cpu().numpy()
    fs = res[0][1][0]
    rel = np.linalg.norm(fs - f1, axis=1) / np.linalg.norm(f1, axis=1)
    assert rel.max() <= 1e-12, rel.max()


def test_bench_launches_its_own_ranks():
    env = dict(os.environ, BD_BENCH_GLOO="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--particles", "16384", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True,
                       timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["parallelism"].startswith("allpairs-shard2")
    assert r.stderr.count("communicator up") == 2, r.stderr[-3000:]
