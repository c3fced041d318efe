"""Launch helper for the method-boundary entry points (include/bd_b200.h,
"method boundary"; csrc/bd_ops.cuh).

The reference's triangulation methods and dynamics functions take numpy
arrays (positions, previous positions, crossings, pair lists) and act on the
triangulation in place.  `OpState` stages such arguments into device
tensors, points a bd_state_t at them and at the triangulation's own device
arrays, launches one op and reads back its small result array.  Each call
synchronises once (for the result), like the reference's methods return
their value.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._lib import check, lib, require_cuda

TRI_KEYS = ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")


def stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def tri_struct(tensors: dict, nv: int) -> _abi.BdTri:
    return _abi.BdTri(nv, int(tensors["edge_v"].shape[0]), int(tensors["tri_v"].shape[0]),
                      *[tensors[k].data_ptr() for k in TRI_KEYS])


def as_device(value, dtype, device, shape=None):
    """numpy array / sequence / tensor -> contiguous device tensor of `dtype`."""
    import torch
    if isinstance(value, torch.Tensor):
        t = value.to(device=device, dtype=dtype)
    else:
        np_dtype = {torch.float64: np.float64, torch.int64: np.int64, torch.uint8: np.uint8}[dtype]
        t = torch.from_numpy(np.ascontiguousarray(value, dtype=np_dtype)).to(device)
    t = t.contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        t = t.reshape(shape)
    return t


class OpState:
    """A bd_state_t + params + workspace for one-shot ops on `n` particles,
    optionally bound to a triangulation (device arrays used in place)."""

    def __init__(self, n: int, L: float, device, tri=None, n_pairs: int = 0, sigma: float = 1.0,
                 tol: float = 1e-12):
        torch = require_cuda()
        self.n = int(n)
        self.device = device
        p = _abi.BdParams()
        p.n = self.n
        p.L = float(L)
        p.sigma = float(sigma)
        p.cap = 0.25 * float(sigma)
        p.clamp = 3.0
        p.tol = float(tol)
        p.max_overlap_iters, p.max_rollbacks = 1000, 10
        lib().bd_prepare_params(ctypes.byref(p))
        p.ncx = 0
        p.pair_capacity = int(n_pairs)
        self.p = p
        ne = tri.n_edges if tri is not None else 0
        nt = tri.n_triangles if tri is not None else 0
        wb = lib().bd_workspace_bytes(ctypes.byref(p), ne, nt)
        self.work = torch.zeros(wb // 8 + 64, dtype=torch.int64, device=device)
        self.res = torch.zeros(8, dtype=torch.int64, device=device)
        self.call_t = torch.zeros(1, dtype=torch.int64, device=device)
        s = _abi.BdState()
        if tri is not None:
            s.tri = tri_struct(tri.tensors(), self.n)
        s.call = self.call_t.data_ptr()
        s.work = self.work.data_ptr()
        s.work_bytes = self.work.numel() * 8
        self.s = s
        self._keep = []

    def bind(self, **tensors):
        """Point state fields (pos, prev, force, alpha, mu, image,
        overlap_flags, pair_a, pair_b) at device tensors."""
        for k, t in tensors.items():
            setattr(self.s, k, t.data_ptr() if t is not None else None)
            self._keep.append(t)
        return self

    def run(self, name: str, *args) -> np.ndarray:
        """Launch lib().name(&state, &params, *args, stream); returns the
        result words (host) after a synchronisation."""
        self.res.zero_()
        fn = getattr(lib(), name)
        check(fn(ctypes.byref(self.s), ctypes.byref(self.p), *args, stream()), name)
        return self.res.cpu().numpy()

    @property
    def res_ptr(self):
        return ctypes.c_void_p(self.res.data_ptr())
