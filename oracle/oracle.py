"""ctypes front-end of the CPU oracle -- TEST INFRASTRUCTURE, NOT THE PRODUCT.

Loads oracle/_build/libbd_oracle.so (oracle/bd_oracle.c, a plain-C
restatement of the reference brownsim hot path).  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this module; the product package never does.

`OracleSim` mirrors the reference's step loops:
  mode "tri"    -> LongRangeSimulation.step (dynamics.py:191-274) with the
                   force model force_mode 0 (long range), 1 (short range over
                   a Verlet list), 2 (long + short), SURVEY.md §0 composites;
  mode "verlet" -> ShortRangeSimulation.step (dynamics.py:326-346);
  mode "abp"    -> AbpSimulation.step (dynamics.py:368-399), see set_abp().
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .noise_np import CounterNormals, normal_pairs  # noqa: F401  (re-export)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libbd_oracle.so")
_lib = None

OK, ERR_SINGULAR, ERR_NONCONV, ERR_STEPFAIL, ERR_FLIP, ERR_NOMEM = 0, 1, 2, 4, 5, 6
RESOLVE_FRAC = 1.0 - 1e-9


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


class TriStruct(ctypes.Structure):
    _fields_ = [("nv", ctypes.c_int64), ("ne", ctypes.c_int64), ("nt", ctypes.c_int64),
                ("tri_v", ctypes.c_void_p), ("tri_shift", ctypes.c_void_p),
                ("tri_edge", ctypes.c_void_p), ("edge_v", ctypes.c_void_p),
                ("edge_tri", ctypes.c_void_p), ("edge_opp", ctypes.c_void_p)]


class SimStruct(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("L", ctypes.c_double),
                ("sigma", ctypes.c_double), ("dt", ctypes.c_double), ("diffusion", ctypes.c_double),
                ("cap", ctypes.c_double), ("clamp", ctypes.c_double), ("r_cut", ctypes.c_double),
                ("skin", ctypes.c_double), ("tol", ctypes.c_double),
                ("max_overlap_iters", ctypes.c_int64), ("max_rollbacks", ctypes.c_int64),
                ("seed", ctypes.c_uint64), ("stream", ctypes.c_uint64), ("call", ctypes.c_uint64),
                ("force_mode", ctypes.c_int64), ("threads", ctypes.c_int64),
                ("pos", ctypes.c_void_p), ("prev", ctypes.c_void_p), ("force", ctypes.c_void_p),
                ("alpha", ctypes.c_void_p), ("mu", ctypes.c_void_p), ("image", ctypes.c_void_p),
                ("overlap_flags", ctypes.c_void_p), ("tri", TriStruct),
                ("vl_np", ctypes.c_int64), ("vl_cap", ctypes.c_int64), ("vl_valid", ctypes.c_int64),
                ("rebuilds", ctypes.c_int64), ("vl_a", ctypes.c_void_p), ("vl_b", ctypes.c_void_p),
                ("vl_snap", ctypes.c_void_p), ("r_list", ctypes.c_double),
                ("disp", ctypes.c_void_p), ("flags_tmp", ctypes.c_void_p), ("cross", ctypes.c_void_p)]


class StatsStruct(ctypes.Structure):
    _fields_ = [("dt_used", ctypes.c_double), ("overlap_iterations", ctypes.c_int64),
                ("flip_passes", ctypes.c_int64), ("inversion_repairs", ctypes.c_int64),
                ("rollbacks", ctypes.c_int64), ("n_overlapping", ctypes.c_int64),
                ("status", ctypes.c_int64), ("err_i", ctypes.c_int64), ("err_k", ctypes.c_int64)]


def _declare(L):
    vp, i64, u64, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    L.bdo_normals.argtypes = [u64, u64, u64, u64, i64, vp]
    L.bdo_long_range.argtypes = [vp, vp, vp, i64, d, ctypes.c_int, vp, vp]
    L.bdo_short_range.argtypes = [vp, vp, vp, i64, vp, vp, i64, d, d, vp, vp]
    L.bdo_overlap_pass.argtypes = [vp, i64, vp, vp, i64, d, d, d, vp, vp]
    L.bdo_overlap_pass.restype = i64
    L.bdo_max_sq_disp.argtypes = [vp, vp, i64, d]
    L.bdo_max_sq_disp.restype = d
    L.bdo_cell_count.argtypes = [d, d]
    L.bdo_cell_count.restype = i64
    L.bdo_cell_grid.argtypes = [vp, i64, d, i64, vp, vp]
    L.bdo_cell_pairs.argtypes = [vp, vp, vp, i64, d, d, vp, vp]
    L.bdo_cell_pairs.restype = i64
    L.bdo_brute_pairs.argtypes = [vp, i64, d, d, vp, vp]
    L.bdo_brute_pairs.restype = i64
    L.bdo_tri_apply_crossings.argtypes = [vp, vp, i64]
    L.bdo_tri_edge_inversion.argtypes = [vp, vp, vp, d]
    L.bdo_tri_edge_inversion.restype = ctypes.c_int
    L.bdo_tri_area2.argtypes = [vp, vp, d, vp]
    L.bdo_tri_delaunay_flags.argtypes = [vp, vp, d, d, vp]
    L.bdo_tri_inverted_flags.argtypes = [vp, vp, d, vp]
    L.bdo_tri_flip.argtypes = [vp, i64]
    L.bdo_tri_flip.restype = ctypes.c_int
    L.bdo_tri_restore_delaunay.argtypes = [vp, vp, d, d, i64]
    L.bdo_tri_restore_delaunay.restype = i64
    L.bdo_tri_repair_inversions.argtypes = [vp, vp, vp, d, i64, vp]
    L.bdo_tri_repair_inversions.restype = ctypes.c_int
    L.bdo_sim_step_tri.argtypes = [vp, vp]
    L.bdo_sim_step_tri.restype = ctypes.c_int
    L.bdo_sim_step_verlet.argtypes = [vp, vp, d]
    L.bdo_sim_step_verlet.restype = ctypes.c_int
    L.bdo_sim_step_abp.argtypes = [vp, vp, vp, d, d, ctypes.c_int, d]
    L.bdo_sim_step_abp.restype = ctypes.c_int
    L.bdo_sim_alloc_scratch.argtypes = [vp]
    L.bdo_sim_free_scratch.argtypes = [vp]
    L.bdo_sim_struct_size.restype = i64
    L.bdo_stats_struct_size.restype = i64
    L.bdo_tri_struct_size.restype = i64
    assert L.bdo_sim_struct_size() == ctypes.sizeof(SimStruct)
    assert L.bdo_stats_struct_size() == ctypes.sizeof(StatsStruct)
    assert L.bdo_tri_struct_size() == ctypes.sizeof(TriStruct)


def _p(a: np.ndarray):
    return a.ctypes.data


# ---------------------------------------------------------------------------
# kernel-level oracles (mirror brownsim._kernels signatures)

def long_range(pos, alpha, mu, L, threads=0):
    pos = np.ascontiguousarray(pos, np.float64)
    n = pos.shape[0]
    out = np.empty((n, 2))
    err = np.empty(n, np.int64)
    lib().bdo_long_range(_p(pos), _p(np.ascontiguousarray(alpha, np.float64)),
                         _p(np.ascontiguousarray(mu, np.float64)), n, float(L), int(threads),
                         _p(out), _p(err))
    return out, err


def short_range(pos, alpha, mu, pa, pb, L, rc):
    pos = np.ascontiguousarray(pos, np.float64)
    n = pos.shape[0]
    pa = np.ascontiguousarray(pa, np.int64)
    pb = np.ascontiguousarray(pb, np.int64)
    out = np.empty((n, 2))
    err = np.empty(n, np.int64)
    lib().bdo_short_range(_p(pos), _p(np.ascontiguousarray(alpha, np.float64)),
                          _p(np.ascontiguousarray(mu, np.float64)), n, _p(pa), _p(pb), pa.size,
                          float(L), float(rc), _p(out), _p(err))
    return out, err


def overlap_pass(pos, pa, pb, L, sigma, resolve=RESOLVE_FRAC):
    pos = np.ascontiguousarray(pos, np.float64)
    n = pos.shape[0]
    pa = np.ascontiguousarray(pa, np.int64)
    pb = np.ascontiguousarray(pb, np.int64)
    disp = np.empty((n, 2))
    flags = np.empty(n, np.uint8)
    c = lib().bdo_overlap_pass(_p(pos), n, _p(pa), _p(pb), pa.size, float(L), float(sigma),
                               float(resolve), _p(disp), _p(flags))
    return disp, flags.astype(bool), int(c)


def max_sq_disp(pos, snap, L):
    pos = np.ascontiguousarray(pos, np.float64)
    snap = np.ascontiguousarray(snap, np.float64)
    return lib().bdo_max_sq_disp(_p(pos), _p(snap), pos.shape[0], float(L))


def cell_grid(pos, L, cell_edge):
    """(ncx, order, cell_start) or None when fewer than 3 cells fit (forces.py:81-99)."""
    pos = np.ascontiguousarray(pos, np.float64)
    ncx = lib().bdo_cell_count(float(L), float(cell_edge))
    if ncx == 0:
        return None
    order = np.empty(pos.shape[0], np.int64)
    cs = np.empty(ncx * ncx + 1, np.int64)
    lib().bdo_cell_grid(_p(pos), pos.shape[0], float(L), ncx, _p(order), _p(cs))
    return ncx, order, cs


def verlet_pairs(pos, L, r_list):
    """build_verlet pair arrays (forces.py:120-142)."""
    pos = np.ascontiguousarray(pos, np.float64)
    g = cell_grid(pos, L, r_list)
    if g is None:
        k = lib().bdo_brute_pairs(_p(pos), pos.shape[0], float(L), float(r_list), None, None)
        pa = np.empty(k, np.int64)
        pb = np.empty(k, np.int64)
        lib().bdo_brute_pairs(_p(pos), pos.shape[0], float(L), float(r_list), _p(pa), _p(pb))
        return pa, pb
    ncx, order, cs = g
    k = lib().bdo_cell_pairs(_p(pos), _p(order), _p(cs), ncx, float(L), float(r_list), None, None)
    pa = np.empty(k, np.int64)
    pb = np.empty(k, np.int64)
    lib().bdo_cell_pairs(_p(pos), _p(order), _p(cs), ncx, float(L), float(r_list), _p(pa), _p(pb))
    return pa, pb


# ---------------------------------------------------------------------------
# triangulation

class OracleTri:
    """The reference PeriodicTriangulation arrays (triangulation.py:129-139),
    maintained by the C restatement."""

    def __init__(self, n_vertices, tri_v, tri_shift, tri_edge, edge_v, edge_tri, edge_opp, L, tol=1e-12):
        self.n_vertices = int(n_vertices)
        self.tri_v = np.ascontiguousarray(tri_v, np.int32).copy()
        self.tri_shift = np.ascontiguousarray(tri_shift, np.int8).copy()
        self.tri_edge = np.ascontiguousarray(tri_edge, np.int32).copy()
        self.edge_v = np.ascontiguousarray(edge_v, np.int32).copy()
        self.edge_tri = np.ascontiguousarray(edge_tri, np.int32).copy()
        self.edge_opp = np.ascontiguousarray(edge_opp, np.int8).copy()
        self.L = float(L)
        self.tol = float(tol)

    @classmethod
    def from_arrays(cls, arrays: dict, n, L):
        return cls(n, arrays["tri_v"], arrays["tri_shift"], arrays["tri_edge"], arrays["edge_v"],
                   arrays["edge_tri"], arrays["edge_opp"], L)

    def arrays(self):
        return {k: getattr(self, k) for k in
                ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")}

    def struct(self):
        return TriStruct(self.n_vertices, self.edge_v.shape[0], self.tri_v.shape[0],
                         _p(self.tri_v), _p(self.tri_shift), _p(self.tri_edge), _p(self.edge_v),
                         _p(self.edge_tri), _p(self.edge_opp))

    def apply_crossings(self, crossings):
        c = np.ascontiguousarray(crossings, np.int64)
        s = self.struct()
        lib().bdo_tri_apply_crossings(ctypes.byref(s), _p(c), c.shape[0])

    def edge_inversion_present(self, prev, curr):
        s = self.struct()
        return bool(lib().bdo_tri_edge_inversion(ctypes.byref(s), _p(np.ascontiguousarray(prev, np.float64)),
                                                 _p(np.ascontiguousarray(curr, np.float64)), self.L))

    def signed_area2(self, pos):
        out = np.empty(self.tri_v.shape[0])
        s = self.struct()
        lib().bdo_tri_area2(ctypes.byref(s), _p(np.ascontiguousarray(pos, np.float64)), self.L, _p(out))
        return out

    def delaunay_flags(self, pos, tol=None):
        out = np.empty(self.edge_v.shape[0], np.uint8)
        s = self.struct()
        lib().bdo_tri_delaunay_flags(ctypes.byref(s), _p(np.ascontiguousarray(pos, np.float64)), self.L,
                                     self.tol if tol is None else float(tol), _p(out))
        return out.astype(bool)

    def inverted_edge_flags(self, pos):
        out = np.empty(self.edge_v.shape[0], np.uint8)
        s = self.struct()
        lib().bdo_tri_inverted_flags(ctypes.byref(s), _p(np.ascontiguousarray(pos, np.float64)), self.L, _p(out))
        return out.astype(bool)

    def flip_edge(self, e):
        s = self.struct()
        rc = lib().bdo_tri_flip(ctypes.byref(s), int(e))
        if rc:
            raise RuntimeError(f"edge {e} not flippable")

    def restore_delaunay(self, pos, tol=None, max_passes=1000):
        s = self.struct()
        r = lib().bdo_tri_restore_delaunay(ctypes.byref(s), _p(np.ascontiguousarray(pos, np.float64)), self.L,
                                           self.tol if tol is None else float(tol), int(max_passes))
        if r < 0:
            raise RuntimeError(f"restore_delaunay failed ({-r})")
        return int(r)

    def repair_inversions(self, pos, prev=None, max_passes=10):
        s = self.struct()
        out = np.zeros(3, np.int64)
        prv = None if prev is None else np.ascontiguousarray(prev, np.float64)
        rc = lib().bdo_tri_repair_inversions(ctypes.byref(s), _p(np.ascontiguousarray(pos, np.float64)),
                                             None if prv is None else _p(prv), self.L, int(max_passes), _p(out))
        if rc:
            raise RuntimeError(f"repair_inversions failed ({rc})")
        return int(out[0]), int(out[1]), bool(out[2])

    def canonical_edge_keys(self):
        """triangulation.py:484-496"""
        sh = self.tri_shift.astype(np.int64)
        tl = self.edge_tri[:, 0]
        ol = self.edge_opp[:, 0].astype(np.int64)
        off = sh[tl, (ol + 2) % 3] - sh[tl, (ol + 1) % 3]
        keys = set()
        for e in range(self.edge_v.shape[0]):
            va, vb = int(self.edge_v[e, 0]), int(self.edge_v[e, 1])
            o = (int(off[e, 0]), int(off[e, 1]))
            keys.add(min((va, vb, o), (vb, va, (-o[0], -o[1]))))
        return keys


# ---------------------------------------------------------------------------
# whole-step oracle

class OracleSim:
    """State + step loop of the reference (see module docstring)."""

    def __init__(self, positions, alpha, mu, L, *, sigma=1.0, dt=0.01, diffusion=0.01,
                 tri: OracleTri | None = None, mode="tri", force_mode=0, r_cutoff=None, skin=None,
                 seed=0, stream=2, call=0, max_overlap_iters=1000, max_rollbacks=10,
                 displacement_cap=None, noise_clamp=3.0, threads=0, track_images=True):
        self.pos = np.ascontiguousarray(positions, np.float64).copy()
        n = self.pos.shape[0]
        self.n = n
        self.prev = self.pos.copy()
        self.force = np.zeros((n, 2))
        self.alpha = np.ascontiguousarray(alpha, np.float64).copy()
        self.mu = np.ascontiguousarray(mu, np.float64).copy()
        self.image = np.zeros((n, 2), np.int64)
        self.overlap_flags = np.zeros(n, np.uint8)
        self.tri = tri
        self.mode = mode
        self.L = float(L)
        skin = 0.5 * sigma if skin is None else float(skin)
        self.skin = skin
        rc = 0.0 if r_cutoff is None else float(r_cutoff)
        self.r_list = max(rc, sigma) + skin
        self.overlap_margin = sigma + skin
        s = SimStruct()
        s.n, s.L = n, self.L
        s.sigma, s.dt, s.diffusion = float(sigma), float(dt), float(diffusion)
        s.cap = sigma / 4.0 if displacement_cap is None else float(displacement_cap)
        s.clamp, s.r_cut, s.skin, s.tol = float(noise_clamp), rc, skin, 1e-12
        s.max_overlap_iters, s.max_rollbacks = int(max_overlap_iters), int(max_rollbacks)
        s.seed, s.stream, s.call = int(seed), int(stream), int(call)
        s.force_mode, s.threads = int(force_mode), int(threads)
        s.pos, s.prev, s.force = _p(self.pos), _p(self.prev), _p(self.force)
        s.alpha, s.mu = _p(self.alpha), _p(self.mu)
        s.image = _p(self.image) if track_images else None
        s.overlap_flags = _p(self.overlap_flags)
        if tri is not None:
            s.tri = tri.struct()
        s.r_list = self.r_list
        self._s = s
        if lib().bdo_sim_alloc_scratch(ctypes.byref(s)):
            raise MemoryError("oracle scratch")

    def __del__(self):
        try:
            lib().bdo_sim_free_scratch(ctypes.byref(self._s))
        except Exception:
            pass

    @property
    def call(self):
        return self._s.call

    @property
    def rebuilds(self):
        return self._s.rebuilds

    def set_abp(self, angles, speed, rot_diffusion, clamp_angle=False, skin=None):
        """mode "abp": AbpSimulation.step (dynamics.py:349-399); r_list =
        overlap_margin = sigma + skin."""
        self.mode = "abp"
        self.angles = np.ascontiguousarray(angles, np.float64).copy()
        self.abp = (float(speed), float(rot_diffusion), int(bool(clamp_angle)))
        self.r_list = self._s.sigma + self.skin
        self.overlap_margin = self.r_list
        self._s.r_list = self.r_list
        self._s.r_cut = 0.0
        return self

    def step(self) -> dict:
        st = StatsStruct()
        if self.mode == "abp":
            lib().bdo_sim_step_abp(ctypes.byref(self._s), ctypes.byref(st), _p(self.angles), *self.abp,
                                   self.overlap_margin)
        elif self.mode == "tri":
            lib().bdo_sim_step_tri(ctypes.byref(self._s), ctypes.byref(st))
        else:
            lib().bdo_sim_step_verlet(ctypes.byref(self._s), ctypes.byref(st), self.overlap_margin)
        return {k: getattr(st, k) for k, _ in StatsStruct._fields_}

    def run(self, steps):
        out = []
        for _ in range(steps):
            st = self.step()
            out.append(st)
            if st["status"]:
                break
        return out

    def unwrapped(self):
        return self.pos + self.image * self.L
