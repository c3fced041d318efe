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
    work = torch.empty(lib().bd_long_range_workspace_bytes(n) // 8 + 8, dtype=torch.int64, device=pos_t.device)
    prec = _abi.BD_LR_FAST if precision == "fast" else _abi.BD_LR_EXACT
    check(lib().bd_long_range_forces(pos_t.data_ptr(), a_t.data_ptr(), m_t.data_ptr(), n, float(L), 0, n, prec,
                                     out.data_ptr(), err.data_ptr(), work.data_ptr(), _stream()),
          "bd_long_range_forces")
    return out.cpu().numpy(), err.cpu().numpy()


def normals(seed: int, stream: int, call: int, n_pairs: int, purpose: int = 0) -> np.ndarray:
    """(n_pairs, 2) counter-based standard normals of one call."""
    torch = require_cuda()
    out = torch.empty((n_pairs, 2), dtype=torch.float64, device="cuda")
    check(lib().bd_normals(seed, stream, call, purpose, n_pairs, out.data_ptr(), _stream()), "bd_normals")
    return out.cpu().numpy()
