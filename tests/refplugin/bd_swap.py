"""pytest plugin -- TEST INFRASTRUCTURE: run the reference's OWN test files
against the B200 engine ("the reference test files become
parity tests unchanged").

    PYTHONPATH=<brownsim install>:tests/refplugin:<repo> \
        python -m pytest -p bd_swap <reference>/tests/test_forces.py ...

At plugin import (before the test modules are collected) the reference's
hot-path entry points are rebound to this package's device implementations,
through the same module-attribute lookups the reference itself uses:

  brownsim._kernels.long_range_kernel / short_range_kernel /
      overlap_pass_kernel / max_sq_displacement / cell_pairs
      (called as _kernels.X by forces.py:52,143,155,163, dynamics.py:113)
      -> paper_1703_02484_b200.kernels (libbd_b200.so)
  brownsim.dynamics.integrate / correct_overlaps (dynamics.py:73-133; called
      by the step loops as module globals, imported by the tests by name)
      -> paper_1703_02484_b200.dynamics.integrate / correct_overlaps on the
         device; integrate draws the reference rng's own normals
         (rng.normals((n, 2))) and feeds them to bd_integrate_noise
  brownsim.triangulation.PeriodicTriangulation.apply_crossings /
      edge_inversion_present / signed_area2 / delaunay_flags /
      inverted_edge_flags / flip_edge / restore_delaunay / repair_inversions
      (triangulation.py:166-363) -> the device methods (csrc/bd_ops.cuh): the
      reference object's numpy arrays are uploaded, the device op runs, and
      mutated arrays are written back in place.

Exceptions raised by the device path are re-raised as the reference's
classes of the same name (brownsim.core).  brute_force_overlaps (the debug
oracle) and everything off the hot path stay the reference's.  Every call
of a replacement is counted; the counts go to $BD_SWAP_REPORT (JSON) at the
end of the session so the caller can check that the device really ran.
"""

from __future__ import annotations

import collections
import functools
import json
import os

import numpy as np

CALLS = collections.Counter()


def _ref_exc(exc):
    import brownsim.core as RC
    cls = getattr(RC, type(exc).__name__, None)
    if cls is None or not (isinstance(cls, type) and issubclass(cls, Exception)):
        cls = RC.BrownsimError
    return cls(str(exc))


def _counted(name):
    def deco(fn):
        @functools.wraps(fn)
        def w(*a, **k):
            CALLS[name] += 1
            from paper_1703_02484_b200.core import BrownsimError
            try:
                return fn(*a, **k)
            except BrownsimError as exc:
                raise _ref_exc(exc) from exc
        return w
    return deco


def _our_box(ref_box):
    from paper_1703_02484_b200.core import PeriodicBox
    return PeriodicBox(float(ref_box.length))


def _our_sys(ref_sys):
    """A device ParticleSystem holding the reference system's arrays."""
    from paper_1703_02484_b200.core import ParticleSystem
    return ParticleSystem(np.asarray(ref_sys.positions), np.asarray(ref_sys.type_of), np.asarray(ref_sys.alpha),
                          np.asarray(ref_sys.mu), _our_box(ref_sys.box))


TRI_KEYS = ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")


def _our_tri(ref_tri):
    from paper_1703_02484_b200.triangulation import PeriodicTriangulation
    return PeriodicTriangulation(_our_box(ref_tri.box), ref_tri.n_vertices,
                                 **{k: getattr(ref_tri, k) for k in TRI_KEYS}, tol=ref_tri.tol)


def _write_back(ref_tri, tri):
    for k, v in tri.arrays().items():
        getattr(ref_tri, k)[...] = v


def install():
    import brownsim._kernels as K
    import brownsim.dynamics as Dy
    import brownsim.triangulation as T

    from paper_1703_02484_b200 import dynamics as D
    from paper_1703_02484_b200 import kernels as G

    # -- kernel boundary (brownsim._kernels) --------------------------------
    @_counted("long_range_kernel")
    def long_range_kernel(pos, alpha, mu, L, tile):
        return G.long_range_kernel(pos, alpha, mu, float(L), tile)

    @_counted("short_range_kernel")
    def short_range_kernel(pos, alpha, mu, pair_a, pair_b, L, r_cutoff):
        return G.short_range_kernel(pos, alpha, mu, pair_a, pair_b, float(L), float(r_cutoff))

    @_counted("overlap_pass_kernel")
    def overlap_pass_kernel(pos, pair_a, pair_b, L, sigma, resolve_frac):
        return G.overlap_pass_kernel(pos, pair_a, pair_b, float(L), float(sigma), float(resolve_frac))

    @_counted("max_sq_displacement")
    def max_sq_displacement(pos, snapshot, L):
        return G.max_sq_displacement(pos, snapshot, float(L))

    @_counted("cell_pairs")
    def cell_pairs(pos, order, cell_start, ncx, L, r_list):
        # the device build bins the particles itself with build_cell_grid's
        # rule (ncx = floor(L / r_list)), so the grid arrays are not needed
        if int(ncx) != int(np.floor(float(L) / float(r_list))):
            raise AssertionError("bd_swap: cell_pairs called with a grid not built for r_list")
        return G.verlet_pairs(pos, float(L), float(r_list))

    K.long_range_kernel = long_range_kernel
    K.short_range_kernel = short_range_kernel
    K.overlap_pass_kernel = overlap_pass_kernel
    K.max_sq_displacement = max_sq_displacement
    K.cell_pairs = cell_pairs

    # -- dynamics functions ----------------------------------------------------
    @_counted("integrate")
    def integrate(sys, forces, params, rng, dt=None):
        ours = _our_sys(sys)
        cross = D.integrate(ours, np.asarray(forces, dtype=np.float64), params, rng, dt)
        sys.snapshot_prev()
        sys.positions[...] = ours.positions_t.cpu().numpy()
        return cross

    @_counted("correct_overlaps")
    def correct_overlaps(sys, pair_a, pair_b, params, tri=None, flags_out=None):
        ours = _our_sys(sys)
        otri = _our_tri(tri) if tri is not None else None
        try:
            return D.correct_overlaps(ours, pair_a, pair_b, params, otri, flags_out)
        finally:
            sys.positions[...] = ours.positions_t.cpu().numpy()
            if tri is not None:
                _write_back(tri, otri)

    Dy.integrate = integrate
    Dy.correct_overlaps = correct_overlaps

    # -- PeriodicTriangulation methods ----------------------------------------
    def method(name, mutates):
        @_counted("tri." + name)
        def m(self, *a, **k):
            tri = _our_tri(self)
            try:
                return getattr(tri, name)(*a, **k)
            finally:
                if mutates:
                    _write_back(self, tri)
        m.__name__ = name
        return m

    for name, mutates in (("apply_crossings", True), ("edge_inversion_present", False), ("signed_area2", False),
                          ("delaunay_flags", False), ("inverted_edge_flags", False), ("flip_edge", True),
                          ("restore_delaunay", True), ("repair_inversions", True)):
        setattr(T.PeriodicTriangulation, name, method(name, mutates))

    # repair_inversions returns the package's RepairResult; the reference's
    # tests compare fields, which have the same names and meanings


install()


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("BD_SWAP_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump({"calls": dict(CALLS), "exitstatus": int(exitstatus)}, f)
