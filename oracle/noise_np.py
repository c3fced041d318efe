"""Counter-based normal noise in pure numpy -- ORACLE / test infrastructure.

This is the third, independent statement of the noise definition in
DESIGN.md §Noise (the others: oracle/bd_oracle.c and the product's
csrc/bd_noise.cuh).  It exists so that the *reference* package can consume
exactly the normals the GPU draws: an instance of `CounterNormals` is passed
as the reference's duck-typed `rng` argument (the reference only calls
`rng.normals(shape, dtype)`, core.py:131-133 via clamped_normals core.py:151-154).

Definition (per call c of normals(shape)):
  element j of the flattened request belongs to pair p = j // 2, component j % 2;
  for attempt = 0, 1, ...: w = Philox4x64-10(counter=(p, c, attempt, purpose),
  key=(seed, stream)); candidate pairs (w0, w1), (w2, w3); v = (w >> 11) *
  2^-52 - 1 exactly; s = v1*v1 + v2*v2; accept the first with 0 < s < 1;
  z = v * sqrt((-2 * log(s)) / s) with the fdlibm-style log below.
Only + - * / sqrt are used, in a fixed order with no fused multiply-add, so
numpy, gcc -ffp-contract=off and CUDA __d*_rn intrinsics agree bit for bit.
"""

from __future__ import annotations

import numpy as np

_M0 = 0xD2E7470EE14C6C93
_M1 = 0xCA5A826395121157
_W0 = 0x9E3779B97F4A7C15
_W1 = 0xBB67AE8584CAA73B
_LO32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def _mulhilo(a: int, b: np.ndarray):
    """64x64 -> 128 multiply of a constant by a uint64 array, via 32-bit limbs."""
    a_lo = np.uint64(a & 0xFFFFFFFF)
    a_hi = np.uint64(a >> 32)
    b_lo = b & _LO32
    b_hi = b >> _S32
    ll = a_lo * b_lo
    lh = a_lo * b_hi
    hl = a_hi * b_lo
    hh = a_hi * b_hi
    mid = (ll >> _S32) + (lh & _LO32) + (hl & _LO32)
    lo = (ll & _LO32) | ((mid & _LO32) << _S32)
    hi = hh + (lh >> _S32) + (hl >> _S32) + (mid >> _S32)
    return hi, lo


def philox4x64(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x64-10 on uint64 arrays (Random123; numpy's np.random.Philox core)."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64).copy() for x in (c0, c1, c2, c3))
    k0 &= (1 << 64) - 1
    k1 &= (1 << 64) - 1
    with np.errstate(over="ignore"):
        for _ in range(10):
            hi0, lo0 = _mulhilo(_M0, c0)
            hi1, lo1 = _mulhilo(_M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
            k0 = (k0 + _W0) & ((1 << 64) - 1)
            k1 = (k1 + _W1) & ((1 << 64) - 1)
    return c0, c1, c2, c3


def _to_pm1(w: np.ndarray) -> np.ndarray:
    return ((w >> np.uint64(11)).astype(np.int64) - (1 << 52)).astype(np.float64) * 2.0**-52


_LN2_HI = 6.93147180369123816490e-01
_LN2_LO = 1.90821492927058770002e-10
_LG = (6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,
       2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,
       1.479819860511658591e-01)


def log_portable(x: np.ndarray) -> np.ndarray:
    """fdlibm-style natural log for positive normal doubles (no fma)."""
    x = np.asarray(x, dtype=np.float64)
    b = x.view(np.uint64)
    e = ((b >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64) - 1023
    m = ((b & np.uint64(0x000FFFFFFFFFFFFF)) | np.uint64(0x3FF0000000000000)).view(np.float64)
    big = m > 1.4142135623730951
    m = np.where(big, m * 0.5, m)
    e = e + big.astype(np.int64)
    lg1, lg2, lg3, lg4, lg5, lg6, lg7 = _LG
    f = m - 1.0
    s = f / (2.0 + f)
    z = s * s
    w = z * z
    t1 = w * (lg2 + w * (lg4 + w * lg6))
    t2 = z * (lg1 + w * (lg3 + w * (lg5 + w * lg7)))
    R = t2 + t1
    hfsq = 0.5 * f * f
    dk = e.astype(np.float64)
    return dk * _LN2_HI - ((hfsq - (s * (hfsq + R) + dk * _LN2_LO)) - f)


def normal_pairs(seed: int, stream: int, call: int, npairs: int, purpose: int = 0) -> np.ndarray:
    """(npairs, 2) standard normals for pairs 0..npairs-1 of one call."""
    out = np.empty((npairs, 2), dtype=np.float64)
    todo = np.arange(npairs, dtype=np.uint64)
    attempt = 0
    while todo.size:
        w0, w1, w2, w3 = philox4x64(todo, np.full(todo.size, call, np.uint64),
                                    np.full(todo.size, attempt, np.uint64),
                                    np.full(todo.size, purpose, np.uint64), seed, stream)
        done = np.zeros(todo.size, dtype=bool)
        for wa, wb in ((w0, w1), (w2, w3)):
            v1 = _to_pm1(wa)
            v2 = _to_pm1(wb)
            s = v1 * v1 + v2 * v2
            ok = (s > 0.0) & (s < 1.0) & ~done
            if ok.any():
                ss = s[ok]
                f = np.sqrt((-2.0 * log_portable(ss)) / ss)
                idx = todo[ok].astype(np.int64)
                out[idx, 0] = v1[ok] * f
                out[idx, 1] = v2[ok] * f
                done |= ok
        todo = todo[~done]
        attempt += 1
    return out


class CounterNormals:
    """Duck-typed stand-in for the reference's RngStream (`.normals(shape, dtype)`).

    Each call consumes one call index, exactly like one `integrate` attempt
    consumes one (N, 2) block in the reference (dynamics.py:89).
    """

    algorithm = "philox4x64-polar-counter"

    def __init__(self, seed: int, stream: int = 2, call: int = 0):
        self.seed = int(seed)
        self.stream = int(stream)
        self.call = int(call)

    def normals(self, shape, dtype=np.float64):
        shape = (shape,) if isinstance(shape, (int, np.integer)) else tuple(shape)
        count = int(np.prod(shape)) if shape else 1
        pairs = normal_pairs(self.seed, self.stream, self.call, (count + 1) // 2)
        self.call += 1
        flat = pairs.reshape(-1)[:count].astype(dtype, copy=False)
        return flat.reshape(shape) if shape else flat[0]
