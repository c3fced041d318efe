"""GPU-backed drop-ins for the reference kernel module brownsim._kernels.

Same names, arguments and return contracts as _kernels.py (numpy in, new
numpy arrays + `err` sentinels out, never raising), each one call into
libbd_b200.so.  A maintainer can bind them into the reference with

    import brownsim._kernels as K, paper_1703_02484_b200.kernels as G
    K.long_range_kernel = G.long_range_kernel   # etc.

because the reference looks them up as module attributes at call time
(forces.py:52, dynamics.py:113).  Each call uploads its inputs and
downloads its outputs; the device-resident simulation classes
(dynamics.py) avoid those copies entirely.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._lib import check, lib, require_cuda


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(a, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def long_range_kernel(pos, alpha, mu, L, tile=32, precision="exact"):
    """_kernels.long_range_kernel (_kernels.py:26-59); `tile` does not change
    results (accumulation is ascending k per receiver either way)."""
    torch = require_cuda()
    pos_t, a_t, m_t = _dev(pos, np.float64), _dev(alpha, np.float64), _dev(mu, np.float64)
    n = pos_t.shape[0]
    out = torch.empty((n, 2), dtype=torch.float64, device=pos_t.device)
    err = torch.empty(n, dtype=torch.int64, device=pos_t.device)
    prec = {"exact": _abi.BD_LR_EXACT, "fast": _abi.BD_LR_FAST, "fast-sym": _abi.BD_LR_FAST_SYM}[precision]
    work = torch.empty(lib().bd_long_range_workspace_bytes_for(n, prec) // 8 + 8, dtype=torch.int64,
                       device=pos_t.device)
    check(lib().bd_long_range_forces(pos_t.data_ptr(), a_t.data_ptr(), m_t.data_ptr(), n, float(L), 0, n, prec,
                                     out.data_ptr(), err.data_ptr(), work.data_ptr(), _stream()),
          "bd_long_range_forces")
    return out.cpu().numpy(), err.cpu().numpy()


def short_range_kernel(pos, alpha, mu, pair_a, pair_b, L, r_cutoff):
    """_kernels.short_range_kernel (_kernels.py:62-91), bit-exact (per-particle
    gather in ascending pair order)."""
    torch = require_cuda()
    pos_t, a_t, m_t = _dev(pos, np.float64), _dev(alpha, np.float64), _dev(mu, np.float64)
    pa, pb = _dev(pair_a, np.int64), _dev(pair_b, np.int64)
    n, P = pos_t.shape[0], pa.shape[0]
    out = torch.empty((n, 2), dtype=torch.float64, device=pos_t.device)
    err = torch.empty(n, dtype=torch.int64, device=pos_t.device)
    work = torch.empty(lib().bd_pairs_workspace_bytes(n, float(L), 0.0, max(P, 1)) // 8 + 64, dtype=torch.int64,
                       device=pos_t.device)
    check(lib().bd_short_range_forces(pos_t.data_ptr(), a_t.data_ptr(), m_t.data_ptr(), n, pa.data_ptr(),
                                      pb.data_ptr(), P, float(L), float(r_cutoff), out.data_ptr(), err.data_ptr(),
                                      work.data_ptr(), _stream()), "bd_short_range_forces")
    return out.cpu().numpy(), err.cpu().numpy()


def overlap_pass_kernel(pos, pair_a, pair_b, L, sigma, resolve_frac):
    """_kernels.overlap_pass_kernel (_kernels.py:94-125): (disp, flags, count)."""
    torch = require_cuda()
    pos_t = _dev(pos, np.float64)
    pa, pb = _dev(pair_a, np.int64), _dev(pair_b, np.int64)
    n, P = pos_t.shape[0], pa.shape[0]
    disp = torch.empty((n, 2), dtype=torch.float64, device=pos_t.device)
    flags = torch.empty(n, dtype=torch.uint8, device=pos_t.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=pos_t.device)
    work = torch.empty(lib().bd_pairs_workspace_bytes(n, float(L), 0.0, max(P, 1)) // 8 + 64, dtype=torch.int64,
                       device=pos_t.device)
    check(lib().bd_overlap_pass(pos_t.data_ptr(), n, pa.data_ptr(), pb.data_ptr(), P, float(L), float(sigma),
                                float(resolve_frac), disp.data_ptr(), flags.data_ptr(), cnt.data_ptr(),
                                work.data_ptr(), _stream()), "bd_overlap_pass")
    return disp.cpu().numpy(), flags.cpu().numpy().astype(bool), int(cnt.item())


def max_sq_displacement(pos, snapshot, L):
    """_kernels.max_sq_displacement (_kernels.py:128-138)."""
    torch = require_cuda()
    p, s = _dev(pos, np.float64), _dev(snapshot, np.float64)
    out = torch.zeros(1, dtype=torch.float64, device=p.device)
    check(lib().bd_max_sq_displacement(p.data_ptr(), s.data_ptr(), p.shape[0], float(L), out.data_ptr(), _stream()),
          "bd_max_sq_displacement")
    return float(out.item())


def verlet_pairs(pos, L, r_list):
    """build_cell_grid + cell_pairs (forces.py:120-142): the ordered pair list."""
    from .core import PeriodicBox
    from .forces import build_verlet
    vl = build_verlet(_dev(pos, np.float64), PeriodicBox(float(L)), float(r_list), 0.0)
    return vl.pair_a.cpu().numpy(), vl.pair_b.cpu().numpy()


def normals(seed: int, stream: int, call: int, n_pairs: int, purpose: int = 0) -> np.ndarray:
    """(n_pairs, 2) counter-based standard normals of one call."""
    torch = require_cuda()
    out = torch.empty((n_pairs, 2), dtype=torch.float64, device="cuda")
    check(lib().bd_normals(seed, stream, call, purpose, n_pairs, out.data_ptr(), _stream()), "bd_normals")
    return out.cpu().numpy()
