"""Test helpers: build product / oracle simulations from golden records."""

from __future__ import annotations

import numpy as np

from golden_io import STAT_KEYS, init_tri


def product_sim(rec, precision="exact", force=None):
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, PeriodicBox, SimParams
    from paper_1703_02484_b200.dynamics import LongRangeSimulation, ShortRangeSimulation
    from paper_1703_02484_b200.triangulation import PeriodicTriangulation

    n = int(rec["n"])
    box = PeriodicBox(float(rec["L"]))
    sys_ = ParticleSystem(rec["pos0"], np.zeros(n, np.int32), rec["alpha"], rec["mu"], box)
    params = SimParams(n=n, sigma=1.0, dt=float(rec["dt"]), diffusion=0.01, r_cutoff=float(rec["r_cutoff"]))
    if str(rec["mode"]) == "verlet":
        return ShortRangeSimulation(sys_, params, CounterRng(int(rec["seed"]), 2))
    tri = PeriodicTriangulation(box, n, **init_tri(rec))
    fm = {0: "long-range", 1: "short-range", 2: "long+short"}[int(rec["force_mode"])] if force is None else force
    return LongRangeSimulation(sys_, params, CounterRng(int(rec["seed"]), 2), tri=tri, force=fm,
                               precision=precision)


def oracle_sim(rec, **kw):
    from oracle import oracle as O
    n = int(rec["n"])
    L = float(rec["L"])
    tri = O.OracleTri.from_arrays(init_tri(rec), n, L) if str(rec["mode"]) == "tri" else None
    return O.OracleSim(rec["pos0"], rec["alpha"], rec["mu"], L, dt=float(rec["dt"]), tri=tri,
                       mode=str(rec["mode"]), force_mode=int(rec["force_mode"]),
                       r_cutoff=float(rec["r_cutoff"]), seed=int(rec["seed"]), stream=2, **kw)


def stats_row(st) -> list:
    if isinstance(st, dict):
        return [float(st[k]) for k in STAT_KEYS]
    return [float(getattr(st, k)) for k in STAT_KEYS]
