"""Write-through host views (paper_1703_02484_b200/_hostview.py): the
reference mutates its state arrays in place (`sys.positions[...] = x`,
core.py:251, dynamics.py:93; `tri.edge_tri[e, 0] = t` in its corruption
tests), so the numpy copies this package hands out must upload such writes
or refuse them -- never drop them silently.

The CPU tests drive HostView over CPU torch tensors (the same code path as
CUDA tensors); the GPU test goes through ParticleSystem / PeriodicTriangulation
/ AbpState and a simulation step."""

import numpy as np
import pytest
import torch

from paper_1703_02484_b200._hostview import HostView, StaleViewError, Versioned


class Owner(Versioned):
    pass


def make(shape=(5, 2)):
    t = torch.arange(int(np.prod(shape)), dtype=torch.float64).reshape(shape)
    o = Owner()
    return t, o, HostView(t, o, "positions")


def test_item_assignment_and_slices_write_through():
    t, o, v = make()
    v[0] = [10.0, 11.0]
    assert t[0].tolist() == [10.0, 11.0]
    v[:, 1] = -1.0
    assert (t[:, 1] == -1.0).all()
    col = v[:, 0]  # a view of the view stays bound
    col[2] = 99.0
    assert t[2, 0] == 99.0


def test_inplace_operators_and_ufunc_out_write_through():
    t, o, v = make()
    v += 1.0
    assert t[0, 0] == 1.0
    v[1] *= 2.0
    assert t[1].tolist() == [6.0, 8.0]
    np.add(v, 1.0, out=v)
    assert t[0, 0] == 2.0
    np.copyto(v, np.zeros((5, 2)))
    assert (t == 0).all()
    v.fill(3.0)
    assert (t == 3.0).all()


def test_copies_and_results_are_plain_arrays():
    t, o, v = make()
    c = v.copy()
    c[0] = 123.0
    assert t[0, 0] == 0.0
    s = v + 1.0
    assert type(s) is np.ndarray
    s[0] = 5.0
    assert t[0, 0] == 0.0
    assert float(v.sum()) == float(t.sum())


def test_stale_view_raises_instead_of_clobbering():
    t, o, v = make()
    o.bump_version()  # the device state changed (a step ran)
    t[0, 0] = 42.0
    with pytest.raises(StaleViewError):
        v[1] = 0.0
    assert t[0, 0] == 42.0  # the newer device value survived
    fresh = HostView(t, o, "positions")
    fresh[1] = 0.0
    assert t[1].tolist() == [0.0, 0.0]


@pytest.mark.gpu
def test_particle_system_triangulation_and_angles_write_through():
    from golden_io import load
    from helpers import product_sim
    rec = load("lr_c0_n256")
    sim = product_sim(rec)
    L = float(rec["L"])
    p = sim.sys.positions
    moved = [float(p[0, 0]) + 1e-7, float(p[0, 1])]  # small moves: the triangulation must stay valid
    p[0] = moved
    assert sim.sys.positions_t[0].tolist() == moved
    y3 = float(np.asarray(p)[3, 1])
    sim.sys.positions[3, 1] += 1e-7
    assert float(sim.sys.positions_t[3, 1]) == y3 + 1e-7
    sim.sys.positions = np.asarray(sim.sys.positions) + L  # attribute assignment wraps like the constructor
    assert float(sim.sys.positions_t.max()) < L
    et = sim.tri.edge_tri
    old = int(et[0, 0])
    et[0, 0] = old  # write-through of an unchanged value keeps the device array
    assert int(sim.tri.tensors()["edge_tri"][0, 0]) == old
    view = sim.sys.positions
    sim.step()
    with pytest.raises(StaleViewError):
        view[0] = 0.0
    with pytest.raises(Exception):
        sim.sys.positions = np.zeros((3, 2))  # wrong shape


@pytest.mark.gpu
def test_reference_rng_is_refused_with_the_replacement_named():
    from golden_io import load
    from helpers import product_sim
    from paper_1703_02484_b200.core import BrownsimError
    rec = load("lr_c0_n256")
    sim = product_sim(rec)

    class RefRng:  # the reference's RngStream: seed / stream, numpy ziggurat normals
        seed, stream = 7, 2

    from paper_1703_02484_b200.dynamics import LongRangeSimulation
    with pytest.raises(BrownsimError, match=r"CounterRng\(7, 2\)"):
        LongRangeSimulation(sim.sys, sim.params, RefRng(), tri=sim.tri)
