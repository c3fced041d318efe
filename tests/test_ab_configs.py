"""Per-step A/B parity at BASELINE.json's configuration sizes (SURVEY.md
§8(c) parity protocol (1)): the GPU step and the CPU oracle's restatement of
the reference step (oracle/bd_oracle.c, pinned bit-exact to reference-made
fixtures) start from the same state -- positions, the six triangulation
arrays, the noise-call counter -- and run the same steps.

  EXACT   : lockstep, every step bit-equal: the all-pairs / short-range
            forces, positions, the six triangulation arrays, the StepStats
            counters (dynamics.py:42-57) and the noise-call counter.
  FAST-SYM: one step from each state of the EXACT trajectory: per particle
            |dF|/|F| <= 1e-9 and |d(displacement)|/|displacement| <= 1e-9
            (the north star's float64 tolerance), the same canonical edge
            keys (triangulation.py:484-496) and the same counters.

cfg3 (N = 131,072 long range, the benchmarked configuration) starts from the
state after 20 FAST-SYM steps (off the initial lattice); cfg2 (16,384, short
range + triangulation) from the initial state and again after 30 steps;
cfg5 (65,536, long + short range) from the initial state; cfg4 (1,048,576
short range at rho 0.6, seed 1) from the device-built initial
triangulation.  The oracle computes its own forces (its all-pairs loop on
all host threads, ~10 s per cfg3 step).

Reference: LongRangeSimulation.step dynamics.py:191-274, long_range_kernel
_kernels.py:26-59, short_range_kernel _kernels.py:62-91,
canonical_edge_keys triangulation.py:484-496.
"""

import os

import numpy as np
import pytest

from golden_io import STAT_KEYS, TRI_KEYS

pytestmark = pytest.mark.gpu
C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
THREADS = os.cpu_count() or 1
FORCE_MODE = {"long-range": 0, "short-range": 1, "long+short": 2}


class Cfg:
    def __init__(self, n, rho, seed, force, r_cutoff=None, device_build=False):
        from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density
        from paper_1703_02484_b200.initial import InitConfig, init_arrays
        self.n, self.seed, self.force = n, seed, force
        self.r_cutoff = r_cutoff
        self.box = PeriodicBox(box_length_for_density(n, 1.0, rho))
        pos, self.types, self.alpha, self.mu = init_arrays(InitConfig(n=n, box=self.box, sigma=1.0, types=C0,
                                                                      seed=seed))
        from paper_1703_02484_b200.core import wrap
        self.pos0 = wrap(self.box, pos)
        from paper_1703_02484_b200.core import SimParams
        self.params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01, r_cutoff=r_cutoff)
        from paper_1703_02484_b200.triangulation import build_initial
        tri = build_initial(self.pos0, self.box, method="device" if device_build else "host")
        self.state0 = {"pos": self.pos0.copy(), "tri": tri.arrays(), "call": 0}

    def gpu(self, state, precision):
        from paper_1703_02484_b200.core import CounterRng, ParticleSystem
        from paper_1703_02484_b200.dynamics import LongRangeSimulation
        from paper_1703_02484_b200.triangulation import PeriodicTriangulation
        sys_ = ParticleSystem(state["pos"], self.types, self.alpha, self.mu, self.box)
        tri = PeriodicTriangulation(self.box, self.n, **state["tri"])
        return LongRangeSimulation(sys_, self.params, CounterRng(self.seed, 2, state["call"]), tri=tri,
                                   force=self.force, precision=precision)

    def oracle(self, state):
        from oracle import oracle as O
        tri = O.OracleTri.from_arrays(state["tri"], self.n, self.box.length)
        return O.OracleSim(state["pos"], self.alpha, self.mu, self.box.length, tri=tri,
                           force_mode=FORCE_MODE[self.force], r_cutoff=self.r_cutoff, seed=self.seed, stream=2,
                           call=state["call"], threads=THREADS)


def gpu_state(sim):
    return {"pos": sim.sys.positions_t.cpu().numpy().copy(), "tri": sim.tri.arrays(), "call": int(sim.rng.call)}


def oracle_state(o):
    return {"pos": o.pos.copy(), "tri": {k: v.copy() for k, v in o.tri.arrays().items()}, "call": int(o.call)}


def mi(d, L):
    return d - np.floor(d / L + 0.5) * L


def ab_exact_lockstep(cfg, state, steps):
    """`steps` EXACT steps on both sides from `state`; every step bit-equal.
    Returns the list of (state before, oracle stats, oracle state after)."""
    g = cfg.gpu(state, "exact")
    o = cfg.oracle(state)
    out = []
    before = state
    for s in range(steps):
        st = g.step()
        so = o.step()
        assert so["status"] == 0, so
        assert [float(getattr(st, k)) for k in STAT_KEYS] == [float(so[k]) for k in STAT_KEYS], (s, st, so)
        assert np.array_equal(g.sys.forces_t.cpu().numpy(), o.force), f"step {s}: forces"
        assert np.array_equal(g.sys.positions_t.cpu().numpy(), o.pos), f"step {s}: positions"
        arrays = g.tri.arrays()
        for k in TRI_KEYS:
            assert np.array_equal(arrays[k], getattr(o.tri, k)), f"step {s}: {k}"
        assert int(g.rng.call) == int(o.call)
        after = oracle_state(o)
        out.append((before, so, after, o.force.copy()))
        before = after
    return out


def ab_fast_sym(cfg, record):
    """One FAST-SYM step from each recorded state against the oracle's step."""
    from oracle import oracle as O
    L = cfg.box.length
    worst_f = worst_x = 0.0
    for s, (before, so, after, f_exact) in enumerate(record):
        g = cfg.gpu(before, "fast-sym")
        st = g.step()
        f = g.sys.forces_t.cpu().numpy()
        rel_f = np.linalg.norm(f - f_exact, axis=1) / np.linalg.norm(f_exact, axis=1)
        d_g = mi(g.sys.positions_t.cpu().numpy() - before["pos"], L)
        d_o = mi(after["pos"] - before["pos"], L)
        rel_x = np.linalg.norm(d_g - d_o, axis=1) / np.linalg.norm(d_o, axis=1)
        worst_f, worst_x = max(worst_f, rel_f.max()), max(worst_x, rel_x.max())
        assert rel_f.max() <= 1e-9, (s, rel_f.max())
        assert rel_x.max() <= 1e-9, (s, rel_x.max(), int(rel_x.argmax()))
        assert [float(getattr(st, k)) for k in STAT_KEYS] == [float(so[k]) for k in STAT_KEYS], (s, st, so)
        keys_g = O.OracleTri.from_arrays(g.tri.arrays(), cfg.n, L).canonical_edge_keys()
        keys_o = O.OracleTri.from_arrays(after["tri"], cfg.n, L).canonical_edge_keys()
        assert keys_g == keys_o, f"step {s}: edge sets differ in {len(keys_g ^ keys_o)} keys"
    return worst_f, worst_x


def test_cfg3_131k_long_range_exact_bitwise_and_fast_sym_per_step():
    cfg = Cfg(131072, 0.3, 0, "long-range")
    warm = cfg.gpu(cfg.state0, "fast-sym")
    warm.run(20)
    record = ab_exact_lockstep(cfg, gpu_state(warm), 3)
    wf, wx = ab_fast_sym(cfg, record)
    print(f"cfg3 fast-sym vs oracle: max |dF|/|F| {wf:.3e}, max |dx|/|x| {wx:.3e}")


def test_cfg2_16k_short_range_tri_exact_bitwise_and_fast_sym_per_step():
    cfg = Cfg(16384, 0.3, 0, "short-range", r_cutoff=2.5)
    ab_exact_lockstep(cfg, cfg.state0, 10)
    warm = cfg.gpu(cfg.state0, "exact")
    warm.run(30)
    record = ab_exact_lockstep(cfg, gpu_state(warm), 5)
    # the short-range force has one arithmetic on the device: FAST-SYM only
    # changes the (absent) long-range part, so the step must still be bit-equal
    g = cfg.gpu(record[0][0], "fast-sym")
    g.step()
    assert np.array_equal(g.sys.positions_t.cpu().numpy(), record[0][2]["pos"])


def test_cfg5_65k_long_plus_short_exact_bitwise_and_fast_sym_per_step():
    cfg = Cfg(65536, 0.3, 0, "long+short", r_cutoff=2.5)
    record = ab_exact_lockstep(cfg, cfg.state0, 2)
    ab_fast_sym(cfg, record)


def test_cfg4_1m_short_range_dense_device_build_exact_bitwise():
    cfg = Cfg(1048576, 0.6, 1, "short-range", r_cutoff=2.5, device_build=True)
    ab_exact_lockstep(cfg, cfg.state0, 2)
