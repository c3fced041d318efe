"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference package is imported read-only from /root/reference/pkg/src.
Its noise argument (`rng`) is served by oracle.noise_np.CounterNormals, the
counter-based generator that the GPU engine also implements, so the recorded
trajectories are the ones the GPU must reproduce.  Composite force modes
(short-range force, or long+short, with the triangulation as
the overlap neighbour provider) are assembled by rebinding the reference's
own `brownsim.dynamics.long_range_forces` global for the duration of
`LongRangeSimulation.step()` -- the step loop itself is the reference's.

Outputs: tests/golden/*.npz (small; committed).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import brownsim.dynamics as dyn  # noqa: E402
from brownsim import _kernels  # noqa: E402
from brownsim.core import PeriodicBox, SimParams, box_length_for_density  # noqa: E402
from brownsim.dynamics import LongRangeSimulation, ShortRangeSimulation  # noqa: E402
from brownsim.forces import (build_cell_grid, build_verlet, long_range_forces,  # noqa: E402
                             short_range_forces, verlet_needs_rebuild)
from brownsim.initial import InitConfig, init_system  # noqa: E402
from brownsim.triangulation import build_initial  # noqa: E402

from oracle.noise_np import CounterNormals  # noqa: E402

C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
C3 = [(0.5, 3.0, -3.0), (0.5, -3.0, 3.0)]
TRI_KEYS = ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")
STAT_KEYS = ("dt_used", "overlap_iterations", "flip_passes", "inversion_repairs", "rollbacks",
             "n_overlapping")


def tri_arrays(tri):
    return {k: getattr(tri, k).copy() for k in TRI_KEYS}


def tri_hash(tri) -> str:
    h = hashlib.sha256()
    for k in TRI_KEYS:
        h.update(np.ascontiguousarray(getattr(tri, k)).tobytes())
    return h.hexdigest()


def pos_hash(pos) -> str:
    return hashlib.sha256(np.ascontiguousarray(pos, np.float64).tobytes()).hexdigest()


class CompositeSimulation(LongRangeSimulation):
    """Reference LongRangeSimulation with only the force call swapped."""

    def __init__(self, sys_, params, rng, tri, force_mode, skin=None):
        super().__init__(sys_, params, rng, tri=tri)
        self.force_mode = force_mode
        self.skin = 0.5 * params.sigma if skin is None else float(skin)
        self.r_list = max(params.r_cutoff, params.sigma) + self.skin
        self.verlet = None
        self.rebuilds = 0

    def _force(self, sys_, box, tile=32):
        lr = long_range_forces(sys_, box, tile).copy() if self.force_mode == 2 else None
        if self.verlet is None or verlet_needs_rebuild(self.verlet, sys_.positions, box):
            grid = build_cell_grid(sys_.positions, box, self.r_list)
            self.verlet = build_verlet(grid, sys_.positions, box, self.r_list, self.skin)
            self.rebuilds += 1
        short_range_forces(sys_, self.verlet, box, self.params.r_cutoff)
        if lr is not None:
            sys_.forces[...] = lr + sys_.forces
        return sys_.forces

    def step(self):
        orig = dyn.long_range_forces
        dyn.long_range_forces = self._force
        try:
            return super().step()
        finally:
            dyn.long_range_forces = orig


def make_system(n, rho, types, seed):
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    return init_system(InitConfig(n=n, box=box, sigma=1.0, types=types, seed=seed)), box


def run_scenario(name, n, rho, types, seed, steps, mode="tri", force_mode=0, dt=0.01,
                 r_cutoff=2.5, full_every=1):
    sys_, box = make_system(n, rho, types, seed)
    params = SimParams(n=n, sigma=1.0, dt=dt, diffusion=0.01, r_cutoff=r_cutoff)
    rng = CounterNormals(seed, stream=2)
    rec = {
        "n": n, "L": box.length, "rho": rho, "seed": seed, "dt": dt, "r_cutoff": r_cutoff,
        "mode": mode, "force_mode": force_mode,
        "pos0": sys_.positions.copy(), "alpha": sys_.alpha.copy(), "mu": sys_.mu.copy(),
    }
    if mode == "tri":
        tri = build_initial(sys_.positions, box)
        for k, v in tri_arrays(tri).items():
            rec["init_" + k] = v
        if force_mode == 0:
            sim = LongRangeSimulation(sys_, params, rng, tri=tri)
        else:
            sim = CompositeSimulation(sys_, params, rng, tri, force_mode)
    else:
        sim = ShortRangeSimulation(sys_, params, rng)
    stats, phash, thash, calls = [], [], [], []
    pos_steps, pos_idx = [], []
    error = ""
    for s in range(steps):
        try:
            st = sim.step()
        except Exception as exc:  # recorded: the GPU must raise the same class
            error = type(exc).__name__
            break
        stats.append([getattr(st, k) for k in STAT_KEYS])
        phash.append(pos_hash(sim.sys.positions))
        thash.append(tri_hash(sim.tri) if mode == "tri" else "")
        calls.append(rng.call)
        if (s + 1) % full_every == 0 or s == steps - 1:
            pos_steps.append(sim.sys.positions.copy())
            pos_idx.append(s)
    rec["stats"] = np.array(stats, dtype=np.float64).reshape(-1, len(STAT_KEYS))
    rec["pos_hash"] = np.array(phash)
    rec["tri_hash"] = np.array(thash)
    rec["calls"] = np.array(calls, np.int64)
    rec["pos_steps"] = np.array(pos_steps)
    rec["pos_idx"] = np.array(pos_idx, np.int64)
    rec["error"] = error
    rec["final_pos"] = sim.sys.positions.copy()
    if mode == "tri":
        for k, v in tri_arrays(sim.tri).items():
            rec["final_" + k] = v
    if hasattr(sim, "rebuilds"):
        rec["rebuilds"] = sim.rebuilds
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
    print(f"{name}: {len(stats)} steps, error={error!r}, "
          f"mean sweeps={np.mean([s[1] for s in stats]) if stats else 0:.2f}, "
          f"flip passes={np.sum([s[2] for s in stats]) if stats else 0:.0f}, "
          f"rollbacks={np.sum([s[4] for s in stats]) if stats else 0:.0f}")


def kernel_fixtures():
    """Reference kernel outputs on the reference tests' own inputs."""
    rec = {}
    # tests/test_forces.py:118-122: random_system(256, 31.0, seed=2, charged=False)
    rng = np.random.default_rng(2)
    L = 31.0
    pos = rng.uniform(0, L, size=(256, 2))
    alpha = rng.normal(size=256)
    mu = rng.normal(size=256)
    from brownsim.core import wrap
    pos = wrap(PeriodicBox(L), pos)
    out, err = _kernels.long_range_kernel(pos, alpha, mu, L, 32)
    rec.update(lr_pos=pos, lr_alpha=alpha, lr_mu=mu, lr_L=L, lr_out=out, lr_err=err)
    # short range over a cell-grid Verlet list, jammed-ish random state
    rng = np.random.default_rng(11)
    L2 = 24.0
    pos2 = rng.uniform(0, L2, size=(400, 2))
    box2 = PeriodicBox(L2)
    grid = build_cell_grid(pos2, box2, 3.0)
    vl = build_verlet(grid, pos2, box2, 3.0, 0.5, overlap_margin=1.5)
    a2 = rng.normal(size=400)
    m2 = rng.normal(size=400)
    sr, sre = _kernels.short_range_kernel(pos2, a2, m2, vl.pair_a, vl.pair_b, L2, 2.5)
    rec.update(sr_pos=pos2, sr_alpha=a2, sr_mu=m2, sr_L=L2, sr_pa=vl.pair_a, sr_pb=vl.pair_b,
               sr_oa=vl.overlap_a, sr_ob=vl.overlap_b, sr_out=sr, sr_err=sre,
               sr_order=grid.order, sr_cell_start=grid.cell_start, sr_ncx=grid.cells_per_axis)
    disp, flags, count = _kernels.overlap_pass_kernel(pos2, vl.overlap_a, vl.overlap_b, L2, 1.0,
                                                      1.0 - 1e-9)
    rec.update(ov_disp=disp, ov_flags=flags, ov_count=count)
    pos3 = np.mod(pos2 + rng.normal(scale=0.3, size=pos2.shape), L2)
    rec.update(msd_pos=pos3, msd_val=_kernels.max_sq_displacement(pos3, pos2, L2))
    # brute-force (no grid) Verlet order, forces.py:136-141
    small = rng.uniform(0, 8.0, size=(40, 2))
    vls = build_verlet(None, small, PeriodicBox(8.0), 3.0, 0.5)
    rec.update(bf_pos=small, bf_L=8.0, bf_pa=vls.pair_a, bf_pb=vls.pair_b)
    # noise known answers for the counter generator (self-pinned, see test_noise)
    cn = CounterNormals(5, stream=2, call=3)
    rec.update(noise_5_2_3=cn.normals((7, 2)))
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **rec)
    print("kernels.npz written")


def build_fixtures():
    """Reference one-time triangulation build (triangulation.py:514-648):
    the quotient arrays before the clean-up flips, and the final arrays."""
    from brownsim.triangulation import _JITTER_KEY, _build_from_tiling
    rec = {}
    for tag, n, rho, seed in (("a", 256, 0.3, 0), ("b", 1000, 0.6, 1)):
        sys_, box = make_system(n, rho, C0, seed)
        pos = sys_.positions.copy()
        gen = np.random.Generator(np.random.Philox(key=np.array(_JITTER_KEY, dtype=np.uint64)))
        jit = pos + gen.standard_normal((n, 2)) * (1e-9 * box.length)
        pre = _build_from_tiling(jit, box, n, 1, 1e-12)
        fin = build_initial(pos, box)
        rec[f"{tag}_pos"] = pos
        rec[f"{tag}_L"] = box.length
        for k in TRI_KEYS:
            rec[f"{tag}_pre_{k}"] = getattr(pre, k)
            rec[f"{tag}_fin_{k}"] = getattr(fin, k)
    np.savez_compressed(os.path.join(HERE, "build.npz"), **rec)
    print("build.npz written")


def main():
    kernel_fixtures()
    build_fixtures()
    run_scenario("lr_c0_n256", 256, 0.3, C0, 0, 30)
    run_scenario("lr_c3_n512", 512, 0.3, C3, 1, 30)
    run_scenario("lr_rollback_n64", 64, 0.35, [(0.5, 3.0, 3.0), (0.5, -3.0, -3.0)], 0, 3, dt=10.0)
    run_scenario("sr_tri_n512", 512, 0.3, C0, 2, 30, force_mode=1)
    run_scenario("lrsr_tri_n256", 256, 0.3, C0, 3, 20, force_mode=2)
    run_scenario("sr_verlet_n512", 512, 0.6, C0, 4, 30, mode="verlet")
    run_scenario("cfg1_lr_c0_n1024", 1024, 0.3, C0, 0, 100, full_every=25)


if __name__ == "__main__":
    main()
