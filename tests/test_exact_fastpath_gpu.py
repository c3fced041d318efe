"""The EXACT all-pairs kernel evaluates each pair's sqrt and division with
branch-free sequences (bd_allpairs.cuh: sqrt_rn_inrange, div_rn_inrange)
when the warp's operands are in range, and falls back to the library's
sqrt() / '/' otherwise.  Bit-exactness of the EXACT path rests on those
sequences returning the correctly rounded (IEEE) results, i.e. the same
bits as sqrt() and '/': checked here on 2^31 generated operand sets
(random mantissas over the guarded exponent range, exact squares and
quotients and one ulp either side, powers of two, all-ones mantissas, and
the kernel's own num / (r2 sqrt(r2)) shape).  The trajectory-level check is
the EXACT A/B parity against the oracle (test_ab_configs.py,
test_gpu_parity.py)."""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 0x5eed])
def test_branch_free_sqrt_and_division_are_correctly_rounded(seed):
    from paper_1703_02484_b200._lib import lib
    bad = torch.zeros(7, dtype=torch.int64, device="cuda")
    rc = lib().bd_probe_exact_arith(ctypes.c_uint64(seed), 1 << 31, ctypes.c_void_p(bad.data_ptr()), None)
    assert rc == 0
    torch.cuda.synchronize()
    b = bad.cpu().tolist()
    assert b[0] == 0, (f"{b[0]} mismatches (sqrt, a/b, r2 sqrt(r2), num/den: {b[3:]}); first operands bits "
                       f"{b[1] & (2**64 - 1):#x} {b[2] & (2**64 - 1):#x}")


def _exact_vs_oracle(pos, alpha, mu, L):
    import numpy as np
    from oracle import oracle as O
    from paper_1703_02484_b200 import kernels
    ref, rerr = O.long_range(pos, alpha, mu, L)
    out, err = kernels.long_range_kernel(pos, alpha, mu, L, 32, precision="exact")
    assert np.array_equal(err, rerr)
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))


def test_tiled_exact_kernel_bitwise_vs_oracle():
    """N above the warp-per-receiver range: the tiled kernel (branch-free
    groups, self tiles, a partial last tile) against the C oracle."""
    import numpy as np
    rng = np.random.default_rng(11)
    n, L = 9001, 150.0
    _exact_vs_oracle(rng.uniform(0, L, size=(n, 2)), rng.normal(size=n), rng.normal(size=n), L)


def test_tiled_exact_kernel_guards_and_fallbacks():
    """Operands outside the branch-free range take the library path, bit-exact
    all the same: zero and -0 / tiny alphas and mus (per-tile and per-receiver
    numerator guards), a pair 1e-120 apart (r^2 below 2^-400: per-group
    fallback) and a coincident pair (the singularity sentinel)."""
    import numpy as np
    rng = np.random.default_rng(12)
    n, L = 8200, 140.0
    pos = rng.uniform(0, L, size=(n, 2))
    alpha = rng.normal(size=n)
    mu = rng.normal(size=n)
    alpha[[5, 300, 4000]] = [0.0, -0.0, 1e-200]
    mu[[7, 301, 5000]] = [0.0, -0.0, 1e-200]
    pos[6000], pos[6001] = [2e-120, 5.0], [1e-120, 5.0]
    pos[7000] = pos[7001]
    _exact_vs_oracle(pos, alpha, mu, L)
