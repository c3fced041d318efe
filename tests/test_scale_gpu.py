"""Full-size checks (BASELINE.json configs) through size-independent
properties: the oracle cannot follow 131k or 262k particles in test time, so
these check what must hold at any size (SURVEY.md §8(c) parity protocol):

  * reciprocal charges (alpha = mu): sum_i F_i = 0 (momentum conservation of
    the all-pairs force) to rounding, for EXACT, FAST and FAST-SYM;
  * EXACT / FAST / FAST-SYM agree per particle within 1e-9 at cfg3's size;
  * Delaunay validity and excluded volume after every step of cfg3 (long
    range, FAST-SYM) and of a dense short-range system (rho 0.6, 262,144
    particles: the wide step kernels);
  * a run is reproducible bit for bit.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
RESOLVE = 1.0 - 1e-9


def workload(n, rho, types, seed=0):
    from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    pos, t, a, m = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=types, seed=seed))
    return box, pos, t, a, m


def test_momentum_conservation_and_precision_agreement_at_cfg3_size():
    from paper_1703_02484_b200 import kernels
    from paper_1703_02484_b200.core import wrap
    n = 131072
    box, pos, t, _, _ = workload(n, 0.3, C0)
    pos = wrap(box, pos)
    rng = np.random.default_rng(1)
    pos = np.mod(pos + rng.normal(scale=0.05, size=pos.shape), box.length)  # off the lattice
    q = np.where(t == 0, 3.0, -3.0)
    out = {}
    for prec in ("exact", "fast", "fast-sym"):
        f, err = kernels.long_range_kernel(pos, q, q, box.length, precision=prec)  # alpha = mu: reciprocal
        assert not err.any()
        scale = np.abs(f).sum(axis=0)
        assert (np.abs(f.sum(axis=0)) <= 1e-11 * scale).all(), (prec, f.sum(axis=0), scale)
        out[prec] = f
    for prec in ("fast", "fast-sym"):
        rel = np.linalg.norm(out[prec] - out["exact"], axis=1) / np.linalg.norm(out["exact"], axis=1)
        assert rel.max() <= 1e-9, (prec, rel.max())


def _check_state(sim, brute):
    from paper_1703_02484_b200.validation import audit_geometry, brute_overlaps, cell_overlaps
    assert audit_geometry(sim) == (0, 0)
    L = sim.sys.box.length
    ov = brute_overlaps(sim.sys.positions_t, L, RESOLVE)[0] if brute else cell_overlaps(sim.sys.positions_t, L,
                                                                                          RESOLVE)
    assert ov == 0


def test_cfg3_fast_sym_steps_stay_valid_and_reproducible():
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, SimParams
    from paper_1703_02484_b200.dynamics import LongRangeSimulation
    from paper_1703_02484_b200.triangulation import build_initial
    n = 131072
    box, pos, t, a, m = workload(n, 0.3, C0)
    sys_a = ParticleSystem(pos, t, a, m, box)
    tri = build_initial(sys_a.positions, box)
    arrays = tri.arrays()
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01)
    sim = LongRangeSimulation(sys_a, params, CounterRng(0, 2), tri=tri, precision="fast-sym")
    for _ in range(5):
        sim.step()
        _check_state(sim, brute=True)
    # the same 5 steps again from the same state: bit for bit
    from paper_1703_02484_b200.triangulation import PeriodicTriangulation
    sys_b = ParticleSystem(pos, t, a, m, box)
    sim_b = LongRangeSimulation(sys_b, params, CounterRng(0, 2), tri=PeriodicTriangulation(box, n, **arrays),
                                precision="fast-sym")
    sim_b.run(5)
    assert np.array_equal(sim.sys.positions, sim_b.sys.positions)
    assert all(np.array_equal(v, sim_b.tri.arrays()[k]) for k, v in sim.tri.arrays().items())


def test_dense_short_range_262k_wide_kernels_stay_valid():
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, SimParams
    from paper_1703_02484_b200.dynamics import LongRangeSimulation
    from paper_1703_02484_b200.triangulation import build_initial
    n = 262144
    box, pos, t, a, m = workload(n, 0.6, C0, seed=1)
    sys_ = ParticleSystem(pos, t, a, m, box)
    tri = build_initial(sys_.positions, box)
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01, r_cutoff=2.5)
    sim = LongRangeSimulation(sys_, params, CounterRng(1, 2), tri=tri, force="short-range")
    for _ in range(3):
        st = sim.step()
        assert st.rollbacks == 0
        _check_state(sim, brute=False)


def test_fast_sym_at_one_million_particles():
    """FAST-SYM at N = 1,048,576 (the workspace, ~n^2/64 bytes = 18 GB, fits
    HBM): per-particle agreement with the directed FAST kernel (itself
    ~1e-13 from the exact sum) within the 1e-9 tolerance, and Newton's third
    law with reciprocal charges."""
    from paper_1703_02484_b200 import kernels
    n = 1 << 20
    rng = np.random.default_rng(7)
    L = float(np.sqrt(n * np.pi * 0.25 / 0.6))
    pos = rng.uniform(0, L, size=(n, 2))
    q = np.where(rng.random(n) < 0.5, 3.0, -3.0)
    mu = np.where(q > 0, 3.0, -1.5)
    fs, e1 = kernels.long_range_kernel(pos, q, mu, L, precision="fast-sym")
    ff, e2 = kernels.long_range_kernel(pos, q, mu, L, precision="fast")
    assert not e1.any() and not e2.any()
    rel = np.linalg.norm(fs - ff, axis=1) / np.linalg.norm(ff, axis=1)
    assert rel.max() <= 1e-9, rel.max()
    fr, _ = kernels.long_range_kernel(pos, q, q, L, precision="fast-sym")  # alpha = mu: reciprocal
    assert (np.abs(fr.sum(axis=0)) <= 1e-10 * np.abs(fr).sum(axis=0)).all()
