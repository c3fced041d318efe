"""FAST-SYM all-pairs force (csrc/bd_allpairs_sym.cuh): each unordered pair's
r^-3 evaluated once and applied to both directions.  Checked against the
EXACT oracle (bit-identical to _kernels.long_range_kernel) within the
north-star tolerance |dF_i| / |F_i| <= 1e-9, on the circulant's corner
cases (one block, odd / even block counts, partial last tile and block),
for determinism, the singularity sentinel and a maintained trajectory."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REL_TOL = 1e-9


def rel_err(a, b):
    return (np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)).max()


@pytest.mark.parametrize("n", [2, 3, 100, 256, 257, 512, 1000, 3000, 4099, 8192])
def test_fast_sym_matches_exact_oracle(n):
    from oracle import oracle as O
    from paper_1703_02484_b200 import kernels
    rng = np.random.default_rng(n)
    L = float(np.sqrt(n * np.pi * 0.25 / 0.3)) + 3.0
    pos = rng.uniform(0, L, size=(n, 2))
    alpha = rng.normal(size=n)
    mu = rng.normal(size=n)
    ref, rerr = O.long_range(pos, alpha, mu, L)
    out, err = kernels.long_range_kernel(pos, alpha, mu, L, 32, precision="fast-sym")
    assert np.array_equal(err, rerr)
    assert rel_err(out, ref) <= REL_TOL


@pytest.mark.parametrize("n,table", [
    (20000, [(2.0, 1.0), (0.0, 3.0), (-1.0, -2.0)]),     # three alphas, one of them 0
    (9000, [(3.0, 3.0), (-3.0, -1.5)]),                  # c0: the factored path almost everywhere
    (5000, [(-0.0, 1.0), (0.0, 2.0), (1.5, 1.0)]),       # -0 and +0 are different groups
    (4099, [(1.0, 1.0)]),                                # one alpha: every tile factored
])
def test_fast_sym_alpha_groups(n, table):
    """Factored tiles (slots sorted by alpha group: tiles / warps with one
    alpha drop the per-pair charge products) and the mixed tiles at group
    boundaries, against the exact oracle."""
    from oracle import oracle as O
    from paper_1703_02484_b200 import kernels
    rng = np.random.default_rng(n)
    L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
    pos = rng.uniform(0, L, size=(n, 2))
    t = rng.integers(0, len(table), n)
    alpha = np.array([a for a, _ in table])[t]
    mu = np.array([m for _, m in table])[t]
    ref, rerr = O.long_range(pos, alpha, mu, L)
    out, err = kernels.long_range_kernel(pos, alpha, mu, L, precision="fast-sym")
    assert np.array_equal(err, rerr)
    nz = np.linalg.norm(ref, axis=1) > 0
    assert rel_err(out[nz], ref[nz]) <= REL_TOL
    assert np.abs(out[~nz]).max(initial=0.0) <= 1e-12


def test_fast_sym_isolated_image_ties():
    """A few exact half-box pairs in an otherwise random state: only the
    receivers flagged by the coordinate-bucket tie check take the exact
    source-side image (EDGE mode); everything else stays on the fast paths."""
    from oracle import oracle as O
    from paper_1703_02484_b200 import kernels
    n = 6000
    rng = np.random.default_rng(7)
    L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
    pos = rng.uniform(0, L, size=(n, 2))
    for i, j in ((5, 4000), (1234, 77), (2999, 3000), (5998, 10)):
        pos[j, 0] = np.mod(pos[i, 0] + 0.5 * L, L)   # x exactly half a box apart
    pos[4500, 1] = np.mod(pos[17, 1] - 0.5 * L, L)    # and one in y
    t = rng.integers(0, 2, n)
    alpha, mu = np.where(t == 0, 3.0, -3.0), np.where(t == 0, 3.0, -1.5)
    ref, rerr = O.long_range(pos, alpha, mu, L)
    out, err = kernels.long_range_kernel(pos, alpha, mu, L, precision="fast-sym")
    assert np.array_equal(err, rerr)
    assert rel_err(out, ref) <= REL_TOL


@pytest.mark.parametrize("name", ["cfg1_lr_c0_n1024", "lr_c3_n512"])
def test_fast_sym_lattice_states_with_exact_image_ties(name):
    """init_system's lattice states hold pairs at exactly L/2 (minimum-image
    ties, where the two directions' images are not mirror images)."""
    from golden_io import load
    from oracle import oracle as O
    from paper_1703_02484_b200 import kernels
    rec = load(name)
    L = float(rec["L"])
    ref, rerr = O.long_range(rec["pos0"], rec["alpha"], rec["mu"], L)
    out, err = kernels.long_range_kernel(rec["pos0"], rec["alpha"], rec["mu"], L, precision="fast-sym")
    assert np.array_equal(err, rerr)
    assert rel_err(out, ref) <= REL_TOL


def test_fast_sym_deterministic_and_close_to_fast_at_cfg3_size():
    from paper_1703_02484_b200 import kernels
    n = 131072
    rng = np.random.default_rng(0)
    L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
    pos = rng.uniform(0, L, size=(n, 2))
    t = rng.integers(0, 2, n)
    alpha, mu = np.where(t == 0, 3.0, -3.0), np.where(t == 0, 3.0, -1.5)
    a, ea = kernels.long_range_kernel(pos, alpha, mu, L, precision="fast-sym")
    b, _ = kernels.long_range_kernel(pos, alpha, mu, L, precision="fast-sym")
    assert np.array_equal(a, b)  # fixed summation order
    f, ef = kernels.long_range_kernel(pos, alpha, mu, L, precision="fast")
    assert np.array_equal(ea, ef) and not ea.any()
    assert rel_err(a, f) <= REL_TOL


def test_fast_sym_reference_golden_and_sentinel():
    from golden_io import load
    from paper_1703_02484_b200 import kernels
    k = load("kernels")
    out, err = kernels.long_range_kernel(k["lr_pos"], k["lr_alpha"], k["lr_mu"], float(k["lr_L"]),
                                         precision="fast-sym")
    assert np.array_equal(err, k["lr_err"])
    assert rel_err(out, k["lr_out"]) <= REL_TOL
    pos = np.array([[1.0, 1.0], [3.0, 2.0], [1.0, 1.0], [5.0, 5.0]])
    _, err = kernels.long_range_kernel(pos, np.ones(4), np.ones(4), 10.0, precision="fast-sym")
    _, err_x = kernels.long_range_kernel(pos, np.ones(4), np.ones(4), 10.0, precision="exact")
    assert np.array_equal(err, err_x) and err[0] == 3


def test_fast_sym_step_tolerance_vs_exact():
    """One maintained step (cfg1 golden initial state): positions after a
    FAST-SYM step agree with the EXACT (reference) step within 1e-9."""
    from golden_io import load
    from helpers import product_sim
    rec = load("cfg1_lr_c0_n1024")
    a = product_sim(rec, precision="exact")
    b = product_sim(rec, precision="fast-sym")
    a.step()
    b.step()
    assert np.abs(a.sys.positions - b.sys.positions).max() <= 1e-9
    assert np.array_equal(a.tri.edge_v, b.tri.edge_v)
