"""Step-level error paths of the device drivers (dynamics.py:191-274 with
forces.py:54-58 and dynamics.py:84-86): a pair at zero separation raises
SingularityError naming the pair, a non-finite force raises StepFailure,
and neither step changes the state.  Both the one-CTA driver (N = 256) and
the grid driver (N = 1,024) run the fused check phase
(bd_drivers.cuh: check_and_backup); EXACT and FAST-SYM forces."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("lr_c0_n256", "exact"), ("cfg1_lr_c0_n1024", "exact"), ("cfg1_lr_c0_n1024", "fast-sym"),
         ("lrsr_tri_n256", "exact")]


@pytest.mark.parametrize("name,precision", CASES + [("sr_tri_n512", "exact")])
def test_zero_separation_raises_singularity(name, precision):
    from golden_io import load
    from helpers import product_sim
    from paper_1703_02484_b200.core import SingularityError
    sim = product_sim(load(name), precision=precision)
    sim.sys.positions[20] = np.asarray(sim.sys.positions)[10]  # write-through: particles 10 and 20 coincide
    before = sim.sys.positions_t.cpu().numpy().copy()
    with pytest.raises(SingularityError, match=r"particles (10 and 20|20 and 10)"):
        sim.step()
    assert np.array_equal(sim.sys.positions_t.cpu().numpy(), before)


@pytest.mark.parametrize("name,precision", CASES)
def test_non_finite_force_raises_step_failure(name, precision):
    from golden_io import load
    from helpers import product_sim
    from paper_1703_02484_b200.core import StepFailure
    sim = product_sim(load(name), precision=precision)
    sim.sys.alpha[7] = np.nan  # every receiver's force becomes NaN
    before = sim.sys.positions_t.cpu().numpy().copy()
    tri_before = {k: v.copy() for k, v in sim.tri.arrays().items()}
    with pytest.raises(StepFailure):
        sim.step()
    assert np.array_equal(sim.sys.positions_t.cpu().numpy(), before)
    after = sim.tri.arrays()
    assert all(np.array_equal(after[k], tri_before[k]) for k in tri_before)
