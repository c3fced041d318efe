"""Validation tools on the GPU (not on the hot path).

debug_overlap_scan  -- the reference's O(N^2) oracle run after every step
                       when debug_scan=True (dynamics.py:136-146), as one
                       kernel (bd_brute_overlaps);
audit_geometry      -- the geometric half of PeriodicTriangulation.audit
                       (triangulation.py:386-482) on the device: triangles
                       with non-positive area and in-circle violations,
                       for checking Delaunay validity at every step of
                       large runs without a host copy.
"""

from __future__ import annotations

import ctypes

from ._lib import check, lib, require_cuda
from .core import BrownsimError

RESOLVE_FRAC = 1.0 - 1e-9


class MissedOverlapError(BrownsimError):
    """Debug scan found an overlapping pair the neighbour provider missed."""


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def brute_overlaps(positions_t, L: float, thresh: float):
    """(count, first pair or None) of pairs closer than thresh."""
    torch = require_cuda()
    out = torch.zeros(2, dtype=torch.int64, device=positions_t.device)
    check(lib().bd_brute_overlaps(positions_t.data_ptr(), int(positions_t.shape[0]), float(L), float(thresh),
                                  out.data_ptr(), _stream()), "bd_brute_overlaps")
    cnt, first = (int(v) for v in out.cpu().numpy())
    if cnt == 0:
        return 0, None
    first &= (1 << 64) - 1
    return cnt, (first >> 32, first & 0xFFFFFFFF)


def debug_overlap_scan(sys, params):
    """Raise MissedOverlapError if any pair anywhere is still overlapping."""
    cnt, first = brute_overlaps(sys.positions_t, sys.box.length, params.sigma * RESOLVE_FRAC)
    if cnt:
        raise MissedOverlapError(f"{cnt} overlapping pairs missed by the neighbor provider, first pair {first}")


def audit_geometry(sim) -> tuple:
    """(n_nonpositive_areas, n_incircle_violations) of a simulation's triangulation, on the device."""
    torch = require_cuda()
    out = torch.zeros(2, dtype=torch.int64, device=sim.sys.device)
    check(lib().bd_tri_audit_geometry(ctypes.byref(sim._eng.s), ctypes.byref(sim.bparams),
                                      ctypes.c_void_p(out.data_ptr()), _stream()), "bd_tri_audit_geometry")
    a, c = (int(v) for v in out.cpu().numpy())
    return a, c


def cell_overlaps(positions_t, L: float, thresh: float) -> int:
    """Number of pairs closer than `thresh`, via the device cell-list pair
    build (bd_verlet_build at radius thresh) -- the O(N) form of the debug
    scan for large N (brute force is O(N^2))."""
    from .core import PeriodicBox
    from .forces import build_verlet
    vl = build_verlet(positions_t, PeriodicBox(float(L)), float(thresh), 0.0)
    if vl.n_pairs == 0:
        return 0
    p = positions_t
    d = p[vl.pair_b] - p[vl.pair_a]
    d = d - (d / L + 0.5).floor() * L
    return int(((d * d).sum(1) < thresh * thresh).sum().item())
