"""Small workload for compute-sanitizer (racecheck / memcheck / synccheck):
the flip / overlap kernels and the FAST-SYM pair kernel at small N.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [what]

what = smem   -- k_step_tri_block_smem (single-CTA shared-memory driver), 3 steps of the N=256 golden
       grid   -- k_step_tri_grid (cooperative grid driver; run with BD_BLOCK_MAX_N=0), 3 steps
       sym    -- FAST-SYM all-pairs (k_allpairs_sym, TMA tiles + mbarriers) at N = 2,500
       ops    -- the method-boundary ops (flip, restore_delaunay, correct_overlaps) on the golden scenarios
Prints OK when the results still equal the reference fixtures (the
sanitizer's report is what the caller checks)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def run_steps():
    from golden_io import load, pos_hash
    from helpers import product_sim
    rec = load("lr_c0_n256")
    sim = product_sim(rec)
    for s in range(3):
        sim.step()
        assert pos_hash(sim.sys.positions) == rec["pos_hash"][s], s


def run_sym():
    from paper_1703_02484_b200 import kernels
    rng = np.random.default_rng(0)
    n, L = 2500, 80.0
    pos = rng.uniform(0, L, (n, 2))
    a = np.where(rng.random(n) < 0.5, 3.0, -3.0)
    m = np.where(a > 0, 3.0, -1.5)
    fs, _ = kernels.long_range_kernel(pos, a, m, L, precision="fast-sym")
    ex, _ = kernels.long_range_kernel(pos, a, m, L, precision="exact")
    rel = np.linalg.norm(fs - ex, axis=1) / np.linalg.norm(ex, axis=1)
    assert rel.max() <= 1e-9, rel.max()


def run_ops():
    from golden_io import load
    from paper_1703_02484_b200.core import PeriodicBox
    from paper_1703_02484_b200.triangulation import PeriodicTriangulation
    k = load("lr_c0_n256")
    n, L = int(k["n"]), float(k["L"])
    tri = PeriodicTriangulation(PeriodicBox(L), n, **{x: k["init_" + x] for x in
                                                     ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri",
                                                      "edge_opp")})
    pos = k["pos0"] + np.random.default_rng(1).normal(scale=0.3, size=(n, 2))
    pos = np.mod(pos, L)
    tri.repair_inversions(pos, pos)
    tri.restore_delaunay(pos)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "smem"
    {"smem": run_steps, "grid": run_steps, "sym": run_sym, "ops": run_ops}[what]()
    print("OK", what)
