"""BASELINE.json configs 1, 2, 4, 5 on one B200: throughput + validity.

bench.py measures the headline config (cfg3).  This runs the others through
the public API and prints one JSON line per config:

  cfg1  N=1,024   long-range all-pairs + triangulation, rho 0.3, 100 steps (EXACT: bit-identical to the reference)
  cfg2  N=16,384  short-range (Verlet, r_cut 2.5) + triangulation maintenance, rho 0.3, 100 steps
  cfg4  N=1,048,576 short-range + triangulation at rho 0.6 (seed 1), 20 steps
  cfg5  N=65,536  long+short non-reciprocal (c0) + triangulation, 10^4 steps, MSD(t)

Every step's state is checked on the device: no triangle with area <= 0,
no in-circle violation (Delaunay-valid), no pair closer than sigma(1-1e-9)
(overlap-free; brute force for N <= 131k, cell list above).  value =
particle-steps/s from the device time of the steps (CUDA events around
each step, validation excluded).  cpu_baseline = the C oracle port of the
same step on this host (a bounded sample of steps).

    python tools/run_configs.py [--cfg 1 2 4 5] [--steps S] [--check-every K]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1703_02484_b200.roofline import hbm_peak_gbs, phase_roofline, step_bytes  # noqa: E402

C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
CFGS = {
    1: dict(n=1024, rho=0.3, force="long-range", precision="exact", steps=100, seed=0),
    2: dict(n=16384, rho=0.3, force="short-range", precision="exact", steps=100, seed=0),
    3: dict(n=131072, rho=0.3, force="long-range", precision="fast-sym", steps=1000, seed=0),  # long-run check
    4: dict(n=1048576, rho=0.6, force="short-range", precision="exact", steps=20, seed=1, build="device"),
    5: dict(n=65536, rho=0.3, force="long+short", precision="fast-sym", steps=10000, seed=0),
}
RESOLVE = 1.0 - 1e-9


def build(cfg):
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, PeriodicBox, SimParams, box_length_for_density
    from paper_1703_02484_b200.dynamics import LongRangeSimulation
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    from paper_1703_02484_b200.triangulation import build_initial
    n = cfg["n"]
    box = PeriodicBox(box_length_for_density(n, 1.0, cfg["rho"]))
    pos, types, alpha, mu = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=C0, seed=cfg["seed"]))
    t0 = time.perf_counter()
    sys_ = ParticleSystem(pos, types, alpha, mu, box)
    tri = build_initial(sys_.positions, box, method=cfg.get("build", "host"))
    t_build = time.perf_counter() - t0
    r_cut = None if cfg["force"] == "long-range" else 2.5
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01, r_cutoff=r_cut)
    sim = LongRangeSimulation(sys_, params, CounterRng(cfg["seed"], 2), tri=tri, force=cfg["force"],
                              precision=cfg["precision"])
    return sim, (pos, alpha, mu, tri.arrays(), box), t_build


def check_state(sim, full_overlap_scan: bool):
    from paper_1703_02484_b200.validation import audit_geometry, brute_overlaps, cell_overlaps
    area, circ = audit_geometry(sim)
    L = sim.sys.box.length
    if full_overlap_scan:
        ov, _ = brute_overlaps(sim.sys.positions_t, L, RESOLVE)
    else:
        ov = cell_overlaps(sim.sys.positions_t, L, RESOLVE)
    return area, circ, ov


def oracle_sample(init, cfg, steps, threads):
    """The C oracle port of the reference step on this host: seconds per step."""
    from oracle import oracle as O
    from paper_1703_02484_b200.core import wrap
    pos, alpha, mu, arrays, box = init
    pos = wrap(box, pos)
    n = cfg["n"]
    tri = O.OracleTri.from_arrays(arrays, n, box.length)
    fm = {"long-range": 0, "short-range": 1, "long+short": 2}[cfg["force"]]
    sim = O.OracleSim(pos, alpha, mu, box.length, tri=tri, force_mode=fm, r_cutoff=None if fm == 0 else 2.5,
                      seed=cfg["seed"], stream=2, threads=threads)
    t0 = time.perf_counter()
    k = 0
    for k in range(1, steps + 1):
        st = sim.step()
        if st["status"]:
            break
    return (time.perf_counter() - t0) / max(k, 1), k


def run(cfg_id, args):
    import torch
    cfg = dict(CFGS[cfg_id])
    if args.steps:
        cfg["steps"] = args.steps
    sim, init, t_build = build(cfg)
    n, K = cfg["n"], cfg["steps"]
    every = args.check_every or {1: 1, 2: 1, 3: 1, 4: 1, 5: 10}[cfg_id]
    # overlap scan: brute force O(N^2) up to 16k every check; above that the
    # cell-list scan every check and the brute force every 100 steps up to 131k
    brute_every = 1 if n <= 16384 else (100 if n <= 131072 else 0)
    sim.run(3)  # warm-up (JIT-free, but first-touch / caches)
    torch.cuda.synchronize()
    u0 = sim.sys.unwrapped_positions().clone()
    msd_t = sorted({int(round(v)) for v in np.logspace(0, np.log10(K), 25)} | {K})
    msd = []
    dev_ms, maint_ms, mbytes, bad, checks, work_tot, pairs = 0.0, 0.0, 0, [], 0, {}, 0
    brute_checks = 0
    ne, nt = sim.tri.n_edges, sim.tri.n_triangles
    stats_tot = dict(overlap_iterations=0, flip_passes=0, inversion_repairs=0, rollbacks=0)
    done = 0
    while done < K:
        chunk = min(every - done % every, K - done)
        for nxt in msd_t:
            if nxt > done:
                chunk = min(chunk, nxt - done)
                break
        res = sim.run(chunk)
        done += chunk
        dev_ms += sum(s.step_ms for s in res)
        maint_ms += sum(s.work["t_total_ns"] for s in res) * 1e-6  # the step kernel (O(N) path incl. SR force)
        pairs = int(sim._eng.vl_meta[0].item()) if cfg["force"] != "long-range" else 0
        mbytes += sum(step_bytes(s.work, n, ne, nt, pairs) for s in res)
        for s_ in res:
            for k, v in s_.work.items():
                work_tot[k] = work_tot.get(k, 0) + v
        for s in res:
            for k in stats_tot:
                stats_tot[k] += getattr(s, k)
        if done in msd_t:
            d = sim.sys.unwrapped_positions() - u0
            msd.append([done, float((d * d).sum(1).mean().item())])
        if done % every == 0 or done == K:
            brute = bool(brute_every) and (done % brute_every == 0 or done == K)
            a, c, o = check_state(sim, brute)
            checks += 1
            brute_checks += int(brute)
            if a or c or o:
                bad.append({"step": done, "nonpositive_areas": a, "incircle_violations": c, "overlaps": o})
    value = n * K / (dev_ms * 1e-3)
    cpu = None
    if not args.no_cpu:
        threads = os.cpu_count() or 1
        budget = {1: 5, 2: 3, 3: 1, 4: 1, 5: 1}[cfg_id]
        t_step, k = oracle_sample(init, cfg, budget, threads)
        cpu = {"value": n / t_step, "unit": "particle-steps/s", "cores": threads, "kind": "port",
               "sample": f"C oracle port of the reference step, {k} step(s) from the initial state "
                         f"(all-pairs on {threads} OpenMP threads, the rest serial like the reference)"}
    line = {"config": f"cfg{cfg_id}", "n": n, "rho": cfg["rho"], "force": cfg["force"],
            "precision": cfg["precision"], "steps": K, "value": value, "unit": "particle-steps/s",
            "ms_per_step": dev_ms / K, "valid_every_checked_step": not bad, "checks": checks,
            "check_every": every, "overlap_scan": f"cell-list at every check, brute force O(N^2) at {brute_checks} "
                                                  f"of them" if brute_every != 1 else "brute force O(N^2)",
            "violations": bad[:5],
            "stats_total": stats_tot, "build_s": t_build, "build": cfg.get("build", "host"), "cpu_baseline": cpu,
            "phase_ms": {"force": (dev_ms - maint_ms) / K, "maintain": maint_ms / K},
            "work_per_step": {k: v / K for k, v in work_tot.items()},
            "phases": phase_roofline({k: v / K for k, v in work_tot.items()}, n, ne, nt, pairs),
            "maintain_roofline": {"bound": "hbm", "achieved": mbytes / (maint_ms * 1e-3) / 1e9, "unit": "GB/s",
                                  "peak": hbm_peak_gbs({}), "frac": mbytes / (maint_ms * 1e-3) / 1e9 / hbm_peak_gbs({}),
                                  "bytes_per_step": mbytes / K},
            "msd": msd if cfg_id in (3, 5) else None}
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="+", default=[1, 2, 5, 4])
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--check-every", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    for c in args.cfg:
        run(c, args)


if __name__ == "__main__":
    main()
