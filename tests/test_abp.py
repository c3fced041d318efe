"""AbpSimulation (dynamics.py:349-399) against the reference's own
trajectories (tests/golden/abp.npz, made by tests/golden/make_golden_ops.py
with the counter noise plugged in as the reference's rng).

  oracle  (C restatement, libm cos/sin)               -> bit-exact
  host    (the product's step_abp compiled for CPU)    -> bit-exact
  gpu     (AbpSimulation on the B200)                  -> angles, stats and
          rebuild counts bit-exact; positions per step (A/B: the GPU state
          is re-loaded from the reference's previous step) within 1e-12
          absolute, and free-running within the north-star tolerance 1e-9.
          The only non-reference arithmetic is the device sincos (<= 1 ulp
          from glibc's cos/sin that numpy calls); jammed overlap correction
          amplifies that over many free-running steps.
"""

import ctypes
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "abp.npz"))
CASES = ("dense", "clamped")
POS_TOL_STEP = 1e-12  # absolute, one step from the reference's state (positions O(10))
POS_TOL_RUN = 1e-9    # absolute, free-running trajectory (north-star per-step tolerance) ...
FREE_STEPS = 15       # ... over the first 15 steps: jammed overlap correction (clamped case: rho 0.7,
                      # V0 = 3, ~9 sweeps per step) amplifies a 1-ulp sincos difference chaotically


def case(name):
    return {k.split("/", 1)[1]: G[k] for k in G.files if k.startswith(name + "/")}


@pytest.mark.parametrize("name", CASES)
def test_oracle_abp_bitwise(name):
    from oracle import oracle as O
    c = case(name)
    n = c["pos0"].shape[0]
    sim = O.OracleSim(c["pos0"], np.zeros(n), np.zeros(n), float(c["L"]), dt=0.01, diffusion=float(c["drot"]),
                      mode="verlet", seed=int(c["seed"]), stream=2)
    sim.set_abp(c["angles0"], float(c["v0"]), float(c["drot"]), bool(c["clamp"]))
    for s in range(c["pos"].shape[0]):
        st = sim.step()
        assert st["status"] == 0
        assert np.array_equal(sim.pos, c["pos"][s]), s
        assert np.array_equal(sim.angles, c["angles"][s]), s
        assert [st["overlap_iterations"], st["n_overlapping"]] == c["stats"][s].tolist(), s
        assert sim.rebuilds == int(c["rebuilds"][s]), s
    assert sim.call == int(c["call_end"])


@pytest.mark.parametrize("name", CASES)
def test_host_driver_abp_bitwise(name):
    from paper_1703_02484_b200._abi import BdStats
    from test_hostemu import HostState, load_emu, params_for
    emu = load_emu()
    c = case(name)
    n = c["pos0"].shape[0]
    p = params_for(emu, float(c["L"]), seed=int(c["seed"]), r_cut=0.0, n=n, force_mode=1, pairs=True)
    p.diffusion = float(c["drot"])
    p.abp_speed, p.abp_rot_diffusion, p.abp_clamp_angle = float(c["v0"]), float(c["drot"]), int(c["clamp"])
    h = HostState(emu, {"n": n, "pos0": c["pos0"], "alpha": np.zeros(n), "mu": np.zeros(n)}, p)
    angles = np.ascontiguousarray(c["angles0"], np.float64).copy()
    h.s.angles = angles.ctypes.data
    st = BdStats()
    for s in range(c["pos"].shape[0]):
        emu.bdh_step_abp(ctypes.byref(h.s), ctypes.byref(p), ctypes.byref(st))
        assert st.status == 0
        assert np.array_equal(h.pos, c["pos"][s]), s
        assert np.array_equal(angles, c["angles"][s]), s
        assert [st.overlap_iterations, st.n_overlapping] == c["stats"][s].tolist(), s
        assert int(h.meta[2]) == int(c["rebuilds"][s]), s
    assert int(h.call[0]) == int(c["call_end"])


def product_abp(c):
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, PeriodicBox, SimParams
    from paper_1703_02484_b200.dynamics import AbpSimulation, AbpState
    n = c["pos0"].shape[0]
    sys_ = ParticleSystem(c["pos0"], np.zeros(n, np.int32), np.zeros(n), np.zeros(n), PeriodicBox(float(c["L"])))
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=float(c["drot"]))
    abp = AbpState(angles=c["angles0"], speed=float(c["v0"]), rot_diffusion=float(c["drot"]))
    return AbpSimulation(sys_, params, CounterRng(int(c["seed"]), 2), abp, clamp_angle_noise=bool(c["clamp"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_abp_matches_reference(name):
    c = case(name)
    sim = product_abp(c)
    for s in range(c["pos"].shape[0]):
        st = sim.step()
        assert np.array_equal(sim.abp.angles, c["angles"][s]), s
        if s < FREE_STEPS:
            assert np.abs(sim.sys.positions - c["pos"][s]).max() <= POS_TOL_RUN, s
            assert [st.overlap_iterations, st.n_overlapping] == c["stats"][s].tolist(), s
            assert sim.rebuilds == int(c["rebuilds"][s]), s
    assert sim.rng.call == int(c["call_end"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_abp_per_step_ab(name):
    """Per-step A/B: load the reference's state of step s-1,
    step once, compare with the reference's step s."""
    c = case(name)
    sim = product_abp(c)
    worst = 0.0
    for s in range(c["pos"].shape[0]):
        if s:
            sim.sys.positions = c["pos"][s - 1]
            sim.abp.angles = c["angles"][s - 1]
        sim.step()
        assert np.array_equal(sim.abp.angles, c["angles"][s]), s
        worst = max(worst, float(np.abs(sim.sys.positions - c["pos"][s]).max()))
    assert worst <= POS_TOL_STEP, worst


@pytest.mark.gpu
def test_gpu_abp_reference_closed_forms():
    """tests/test_dynamics.py:288-311: ballistic displacement, frozen
    positions at V0 = 0, straight line of a single particle."""
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, PeriodicBox, SimParams
    from paper_1703_02484_b200.dynamics import AbpSimulation, AbpState
    import math

    def make(pos, L, v0, angles, drot):
        n = len(pos)
        sys_ = ParticleSystem(np.asarray(pos, float), np.zeros(n, np.int32), np.zeros(n), np.zeros(n),
                              PeriodicBox(L))
        params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=drot)
        return AbpSimulation(sys_, params, CounterRng(0, 2), AbpState(np.asarray(angles, float), v0, drot))

    sim = make([[5, 5], [15, 5], [5, 15], [15, 15]], 30.0, 1.0, np.zeros(4), 0.0)
    before = sim.sys.positions.copy()
    sim.step()
    assert np.allclose(sim.sys.positions - before, [[0.01, 0.0]] * 4, atol=1e-14)
    assert np.array_equal(sim.abp.angles, np.zeros(4))
    sim = make([[10.0, 10.0]], 50.0, 1.0, [math.pi / 4], 0.0)
    y0 = sim.sys.positions[0, 1] - sim.sys.positions[0, 0]
    sim.run(100)
    assert abs(sim.sys.positions[0, 1] - sim.sys.positions[0, 0] - y0) < 1e-9
    n = 1024
    rng = np.random.default_rng(0)
    pos = np.stack(np.meshgrid(np.arange(32) * 3.0, np.arange(32) * 3.0), -1).reshape(-1, 2) + 1.0
    sim = make(pos, 96.0, 0.0, np.zeros(n), 0.01)
    sim.run(25)
    assert np.array_equal(sim.sys.positions, pos)  # V0 = 0 freezes positions
    assert sim.abp.angles.var() == pytest.approx(2 * 0.01 * 0.01 * 25, rel=0.1)
    del rng
