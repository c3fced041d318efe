"""Reference-API compatibility of the standalone helpers (brownsim.forces /
core names and signatures): build_cell_grid + build_verlet(grid, ...),
verlet_needs_rebuild on numpy positions, clamped_normals / clamped_gaussian
over the counter noise, and integrate() driven by any rng with the
reference's normals(shape, dtype) method (bd_integrate_noise)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_cell_grid_and_verlet_reference_signatures():
    from golden_io import load
    from oracle import oracle as O
    from paper_1703_02484_b200.core import PeriodicBox
    from paper_1703_02484_b200.forces import build_cell_grid, build_verlet, verlet_needs_rebuild
    k = load("kernels")
    pos, L = k["sr_pos"], float(k["sr_L"])
    box = PeriodicBox(L)
    grid = build_cell_grid(pos, box, 3.0)
    ncx, order, cs = O.cell_grid(pos, L, 3.0)
    assert grid.cells_per_axis == ncx
    assert np.array_equal(grid.order.cpu().numpy(), order) and np.array_equal(grid.cell_start.cpu().numpy(), cs)
    vl = build_verlet(grid, pos, box, 3.0, 0.5, 1.5)  # the reference's argument order
    assert np.array_equal(vl.pair_a.cpu().numpy(), k["sr_pa"]) and np.array_equal(vl.pair_b.cpu().numpy(), k["sr_pb"])
    assert vl.overlap_a is not None
    assert not verlet_needs_rebuild(vl, pos, box)
    moved = pos.copy()
    moved[0] += 0.3  # > skin / 2
    assert verlet_needs_rebuild(vl, np.mod(moved, L), box)
    tiny = PeriodicBox(5.0)
    assert build_cell_grid(np.zeros((3, 2)), tiny, 3.0) is None


def test_counter_normals_and_clamped_helpers():
    from oracle.noise_np import normal_pairs
    from paper_1703_02484_b200.core import CounterRng, clamped_gaussian, clamped_normals
    rng = CounterRng(11, 2)
    z = clamped_normals(rng, (100, 2), clamp=3.0)
    ref = np.clip(normal_pairs(11, 2, 0, 100), -3.0, 3.0)
    assert np.array_equal(z, ref)
    assert rng.call == 1
    g = clamped_gaussian(rng, 0.5)
    assert -0.5 <= g <= 0.5 and rng.call == 2


def test_integrate_with_a_numpy_rng_matches_the_reference_formula():
    """integrate() with the reference's own kind of rng (numpy normals): the
    device consumes the very normals the rng returns (dynamics.py:89-93)."""
    from paper_1703_02484_b200.core import ParticleSystem, PeriodicBox, SimParams, wrap
    from paper_1703_02484_b200.dynamics import integrate

    class NumpyRng:
        def __init__(self, seed):
            self.g = np.random.default_rng(seed)

        def normals(self, shape, dtype=np.float64):
            return self.g.standard_normal(size=shape, dtype=dtype)

    n, L = 500, 40.0
    r0 = np.random.default_rng(3)
    pos = r0.uniform(0, L, (n, 2))
    F = r0.normal(size=(n, 2))
    box = PeriodicBox(L)
    sys_ = ParticleSystem(pos, np.zeros(n, np.int32), np.ones(n), np.ones(n), box)
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01)
    cross = integrate(sys_, F, params, NumpyRng(5))
    xi = np.clip(np.random.default_rng(5).standard_normal(size=(n, 2)), -3.0, 3.0)
    new = (pos + F * 0.01) + xi * np.sqrt(0.01 * 0.01)
    wrapped = wrap(box, new)
    assert np.array_equal(sys_.positions_t.cpu().numpy(), wrapped)
    assert np.array_equal(sys_.positions_prev_t.cpu().numpy(), pos)
    assert np.array_equal(cross, np.rint((new - wrapped) / L).astype(np.int64))
