"""Force models and neighbour structures (mirrors brownsim.forces).

The interaction laws are the reference's (forces.py:23-60, :159-172): the
long-range law f(r) = r / r^3 over all directed pairs and the short-range
law f(r) = r / r^7 truncated at r_cutoff over Verlet half-lists built from a
periodic cell grid.  Here they run on the GPU:

  * long_range_forces / short_range_forces / build_verlet operate on a
    device-resident ParticleSystem through the C ABI (one kernel launch
    each, no host round trip);
  * inside a simulation step the Verlet list lives in HBM and is rebuilt on
    the device when stale (csrc/bd_verlet.cuh), so these helpers are for
    standalone use and validation.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._lib import check, lib, require_cuda
from .core import ConfigError, ParticleSystem, PeriodicBox, SingularityError

LONG_RANGE = "long-range"
SHORT_RANGE = "short-range"


@dataclass(frozen=True)
class ForceLaw:
    """forces.py:23-34"""

    kind: str
    r_cutoff: float | None = None

    def __post_init__(self):
        if self.kind not in (LONG_RANGE, SHORT_RANGE):
            raise ConfigError(f"unknown force kind {self.kind!r}")
        if self.kind == SHORT_RANGE and (self.r_cutoff is None or self.r_cutoff <= 0):
            raise ConfigError("short-range law requires a positive r_cutoff")


def pair_force(law: ForceLaw, mu_i: float, alpha_k: float, r_ik) -> np.ndarray:
    """Force on receiver i from source k (forces.py:37-47), host scalar helper."""
    r_ik = np.asarray(r_ik, dtype=np.float64)
    r = math.sqrt(float(r_ik[0]) ** 2 + float(r_ik[1]) ** 2)
    if r == 0.0:
        raise SingularityError("pair at zero separation")
    if law.kind == LONG_RANGE:
        return mu_i * alpha_k * r_ik / r**3
    if r > law.r_cutoff:
        return np.zeros(2)
    return mu_i * alpha_k * r_ik / r**7


def verlet_pair_capacity(n: int, L: float, r_list: float, sigma: float = 1.0) -> int:
    """Upper bound on the Verlet pairs of n hard disks (diameter sigma) in a
    box of side L: neighbours of a disk within r_list cannot outnumber the
    hexagonal packing of the disk of radius r_list + sigma (area sqrt(3)/2
    sigma^2 per disk), with 1.5x slack for transient overlaps."""
    if n < 2:
        return 1
    per = math.pi * (r_list + sigma) ** 2 / (math.sqrt(3.0) / 2.0 * sigma * sigma)
    bound = int(math.ceil(n * per * 0.5 * 1.5)) + 64
    return int(min(bound, n * (n - 1) // 2 + 1))


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def long_range_forces(sys: ParticleSystem, box: PeriodicBox, tile: int = 32, precision: str = "exact"):
    """All-pairs forces into sys.forces_t (forces.py:50-60); raises SingularityError."""
    torch = require_cuda()
    n = sys.n
    err = torch.empty(n, dtype=torch.int64, device=sys.device)
    work = torch.empty(lib().bd_long_range_workspace_bytes(n) // 8 + 8, dtype=torch.int64, device=sys.device)
    prec = _abi.BD_LR_FAST if precision == "fast" else _abi.BD_LR_EXACT
    check(lib().bd_long_range_forces(sys.positions_t.data_ptr(), sys.alpha_t.data_ptr(), sys.mu_t.data_ptr(), n,
                                     float(box.length), 0, n, prec, sys.forces_t.data_ptr(), err.data_ptr(),
                                     work.data_ptr(), _stream()), "bd_long_range_forces")
    _raise_singular(err)
    return sys.forces_t


def _raise_singular(err):
    bad = (err != 0).nonzero()
    if bad.numel():
        i = int(bad[0, 0].item())
        raise SingularityError(f"particles {i} and {int(err[i].item()) - 1} at zero separation")


@dataclass
class VerletList:
    """Half-list of unordered pairs within r_list + snapshot (forces.py:102-117), in HBM."""

    pair_a: object  # torch int64 (P,)
    pair_b: object
    snapshot: object  # torch float64 (N, 2)
    r_list: float
    skin: float
    overlap_a: object = field(default=None, repr=False)
    overlap_b: object = field(default=None, repr=False)

    @property
    def n_pairs(self) -> int:
        return int(self.pair_a.shape[0])


@dataclass
class CellGrid:
    """Uniform periodic bins (forces.py:67-78): `order` = particle ids sorted
    by cell (stable), `cell_start` = CSR bounds.  Device tensors here."""

    cells_per_axis: int
    cell_edge: float
    order: object  # torch int64 (N,)
    cell_start: object  # torch int64 (ncells + 1,)

    @property
    def n_cells(self) -> int:
        return self.cells_per_axis * self.cells_per_axis


def build_cell_grid(positions, box: PeriodicBox, cell_edge: float):
    """forces.py:81-99: bin wrapped positions into cells of edge >= cell_edge;
    None when fewer than 3 cells fit per axis (the caller pairs by brute
    force).  Computed on the device with the reference's formula (floor,
    clip, stable sort, bincount, cumsum).  build_verlet does its own binning
    in the Verlet kernel and only looks at whether the grid is None."""
    torch = require_cuda()
    ncx = int(math.floor(box.length / cell_edge))
    if ncx < 3:
        return None
    edge = box.length / ncx
    pos = _as_positions(positions)
    ij = torch.floor(pos / edge).to(torch.int64).clamp_(0, ncx - 1)
    cell_id = ij[:, 0] + ij[:, 1] * ncx
    order = torch.sort(cell_id, stable=True).indices
    counts = torch.bincount(cell_id, minlength=ncx * ncx)
    cell_start = torch.zeros(ncx * ncx + 1, dtype=torch.int64, device=pos.device)
    torch.cumsum(counts, 0, out=cell_start[1:])
    return CellGrid(ncx, edge, order, cell_start)


def _as_positions(positions):
    torch = require_cuda()
    if hasattr(positions, "data_ptr"):
        return positions.contiguous()
    return torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float64)).cuda()


def build_verlet(*args, **kwargs) -> VerletList:
    """Every unordered pair within r_list, in the reference's exact order
    (cell scan, forces.py:120-150 / _kernels.py:141-236), built on the GPU.

    Signature of the reference: build_verlet(grid, positions, box, r_list,
    skin, overlap_margin=None); build_verlet(positions, box, r_list, skin,
    overlap_margin=None) is accepted too.  The device kernel bins the
    particles itself, with the same rule as build_cell_grid (fewer than 3
    cells per axis -> np.triu_indices order), so `grid` only has to be
    build_cell_grid's answer for the same positions."""
    if len(args) >= 2 and isinstance(args[1], PeriodicBox):
        positions, box, r_list, skin, *rest = args
    else:
        _grid, positions, box, r_list, skin, *rest = args
    overlap_margin = rest[0] if rest else kwargs.get("overlap_margin")
    torch = require_cuda()
    pos = _as_positions(positions)
    n = int(pos.shape[0])
    L = float(box.length)
    cap = verlet_pair_capacity(n, L, r_list)
    while True:
        pa = torch.empty(cap, dtype=torch.int64, device=pos.device)
        pb = torch.empty(cap, dtype=torch.int64, device=pos.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=pos.device)
        work = torch.empty(lib().bd_pairs_workspace_bytes(n, L, float(r_list), cap) // 8 + 64, dtype=torch.int64,
                           device=pos.device)
        check(lib().bd_verlet_build(pos.data_ptr(), n, L, float(r_list), pa.data_ptr(), pb.data_ptr(), cap,
                                    cnt.data_ptr(), work.data_ptr(), _stream()), "bd_verlet_build")
        k = int(cnt.item())
        if k <= cap:
            break
        cap = k + 64
    vl = VerletList(pa[:k].clone(), pb[:k].clone(), pos.clone(), float(r_list), float(skin))
    if overlap_margin is not None:
        d = pos[vl.pair_b] - pos[vl.pair_a]
        d = d - torch.floor(d / L + 0.5) * L
        near = (d * d).sum(dim=1) <= overlap_margin * overlap_margin
        vl.overlap_a, vl.overlap_b = vl.pair_a[near], vl.pair_b[near]
    return vl


def verlet_needs_rebuild(vl: VerletList, positions, box: PeriodicBox) -> bool:
    """forces.py:153-156 on the GPU (max_sq_displacement kernel); positions
    may be a numpy array or a device tensor."""
    torch = require_cuda()
    pos = _as_positions(positions)
    snap = _as_positions(vl.snapshot)
    out = torch.zeros(1, dtype=torch.float64, device=snap.device)
    check(lib().bd_max_sq_displacement(pos.data_ptr(), snap.data_ptr(), int(pos.shape[0]),
                                       float(box.length), out.data_ptr(), _stream()), "bd_max_sq_displacement")
    return bool(out.item() > (vl.skin / 2.0) ** 2)


def short_range_forces(sys: ParticleSystem, vl: VerletList, box: PeriodicBox, r_cutoff: float):
    """Truncated forces over the Verlet pairs into sys.forces_t (forces.py:159-172)."""
    torch = require_cuda()
    n, P = sys.n, vl.n_pairs
    err = torch.empty(n, dtype=torch.int64, device=sys.device)
    work = torch.empty(lib().bd_pairs_workspace_bytes(n, float(box.length), 0.0, max(P, 1)) // 8 + 64,
                       dtype=torch.int64, device=sys.device)
    check(lib().bd_short_range_forces(sys.positions_t.data_ptr(), sys.alpha_t.data_ptr(), sys.mu_t.data_ptr(), n,
                                      vl.pair_a.data_ptr(), vl.pair_b.data_ptr(), P, float(box.length),
                                      float(r_cutoff), sys.forces_t.data_ptr(), err.data_ptr(), work.data_ptr(),
                                      _stream()), "bd_short_range_forces")
    _raise_singular(err)
    return sys.forces_t
