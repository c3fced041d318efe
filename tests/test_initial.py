"""The one-time initial state (paper_1703_02484_b200/initial.py) equals the
reference's init_system (initial.py:114-130) bit for bit: positions, types,
alpha and mu of every golden scenario were written by the reference itself
(tests/golden/make_golden.py), from the configs listed here."""

import numpy as np
import pytest

from golden_io import load

C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
C3 = [(0.5, 3.0, -3.0), (0.5, -3.0, 3.0)]
CASES = [("lr_c0_n256", 256, 0.3, C0, 0), ("lr_c3_n512", 512, 0.3, C3, 1),
         ("lr_rollback_n64", 64, 0.35, [(0.5, 3.0, 3.0), (0.5, -3.0, -3.0)], 0),
         ("sr_tri_n512", 512, 0.3, C0, 2), ("lrsr_tri_n256", 256, 0.3, C0, 3),
         ("sr_verlet_n512", 512, 0.6, C0, 4), ("cfg1_lr_c0_n1024", 1024, 0.3, C0, 0)]


@pytest.mark.parametrize("name,n,rho,types,seed", CASES, ids=[c[0] for c in CASES])
def test_init_arrays_equal_reference(name, n, rho, types, seed):
    from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    rec = load(name)
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    assert box.length == float(rec["L"])
    pos, _t, alpha, mu = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=types, seed=seed))
    assert np.array_equal(pos, rec["pos0"])
    assert np.array_equal(alpha, rec["alpha"]) and np.array_equal(mu, rec["mu"])


def test_reservoir_sample_matches_algorithm_r():
    from paper_1703_02484_b200.initial import _stream, reservoir_sample
    for pop, k, seed in ((1000, 10, 0), (500, 499, 1), (50, 50, 2), (70, 1, 3)):
        got = reservoir_sample(pop, k, _stream(seed, 1))
        g = _stream(seed, 1)
        res = np.arange(k, dtype=np.int64)
        if 0 < k < pop:
            js = g.integers(0, np.arange(k + 1, pop + 1))
            for i in range(k, pop):  # the reference's loop (initial.py:97-101)
                if js[i - k] < k:
                    res[js[i - k]] = i
        assert np.array_equal(got, np.sort(res))
