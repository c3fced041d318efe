"""Periodic Delaunay triangulation resident in HBM.

PeriodicTriangulation holds the reference's six arrays (triangulation.py:
120-139) as CUDA tensors with the same dtypes and layout; all maintenance
(apply_crossings, pass-through check, inversion repair, Lawson flips) runs
inside the device step (csrc/bd_step.cuh).  Host methods here are for setup,
read-out and validation (audit, canonical_edge_keys), as in the reference.

build_initial() restates the reference's one-time construction
(triangulation.py:514-648: jittered (2m+1)^2 tiling -> scipy Qhull ->
quotient onto the torus) in vectorised numpy so it scales to 1M particles;
its output arrays are identical to the reference's (tests/test_setup_and_abi.py).
The post-build Delaunay clean-up pass runs on the GPU.
build_initial(method="device") builds the triangulation itself on the GPU
(csrc/bd_build.cuh: per-point Voronoi cells by bisector clipping).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._hostview import HostView, Versioned
from .core import BrownsimError, BuildError, NonConvergenceError, PeriodicBox

DEFAULT_TOL = 1e-12
_JITTER_KEY = (0x7C94_1EAF, 0x0B5E_55ED)  # triangulation.py:24 (build jitter must match)
TRI_KEYS = ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")
_DTYPES = {"tri_v": np.int32, "tri_shift": np.int8, "tri_edge": np.int32, "edge_v": np.int32,
           "edge_tri": np.int32, "edge_opp": np.int8}
_SHAPES = {"tri_v": (3,), "tri_shift": (3, 2), "tri_edge": (3,), "edge_v": (2,), "edge_tri": (2,),
           "edge_opp": (2,)}


@dataclass(frozen=True)
class FlipDecision:
    """triangulation.py:27-30"""

    edge: int
    reason: str  # "delaunay-violation" | "inverted-triangle"


@dataclass
class RepairResult:
    """triangulation.py:33-37"""

    flips: int
    passes: int
    needs_rollback: bool


@dataclass
class AuditReport:
    """triangulation.py:40-63"""

    n_vertices: int
    n_edges: int
    n_triangles: int
    euler_ok: bool
    refs_ok: bool
    min_area: float
    n_nonpositive_areas: int
    n_incircle_violations: int
    max_circumdiameter: float
    circumdiameter_ok: bool
    shifts_in_range: bool
    messages: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return (self.euler_ok and self.refs_ok and self.n_nonpositive_areas == 0
                and self.n_incircle_violations == 0)


class PeriodicTriangulation(Versioned):
    """Vertex/edge/triangle arrays with opposite-vertex links on the torus."""

    def __init__(self, box: PeriodicBox, n_vertices: int, tri_v, tri_shift, tri_edge, edge_v, edge_tri,
                 edge_opp, tol: float = DEFAULT_TOL, device=None):
        import torch
        self.box = box
        self.n_vertices = int(n_vertices)
        self.tol = float(tol)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        arrays = dict(tri_v=tri_v, tri_shift=tri_shift, tri_edge=tri_edge, edge_v=edge_v, edge_tri=edge_tri,
                      edge_opp=edge_opp)
        self._t = {}
        for k in TRI_KEYS:
            a = arrays[k]
            if isinstance(a, torch.Tensor):
                t = a.to(dev).contiguous()
            else:
                t = torch.from_numpy(np.ascontiguousarray(a, dtype=_DTYPES[k])).to(dev)
            self._t[k] = t
        # rollback copy (save_state / restore_state, triangulation.py:158-164)
        self._backup = {k: torch.empty_like(v) for k, v in self._t.items()}

    # device tensors
    def tensors(self) -> dict:
        return self._t

    def backup_tensors(self) -> dict:
        return self._backup

    # host copies (numpy, write-through: _hostview.HostView), named like the
    # reference's attributes; `tri.edge_tri[e, 0] = x` reaches the device
    def __getattr__(self, name):
        if name in TRI_KEYS:
            return HostView(self._t[name], self, name)
        raise AttributeError(name)

    def arrays(self) -> dict:
        return {k: v.cpu().numpy() for k, v in self._t.items()}

    def load_arrays(self, arrays: dict):
        import torch
        for k in TRI_KEYS:
            self._t[k].copy_(torch.from_numpy(np.ascontiguousarray(arrays[k], dtype=_DTYPES[k])))
        self.bump_version()

    @property
    def n_triangles(self) -> int:
        return int(self._t["tri_v"].shape[0])

    @property
    def n_edges(self) -> int:
        return int(self._t["edge_v"].shape[0])

    @property
    def edges(self):
        return self.edge_v

    def save_state(self):
        return {k: v.clone() for k, v in self._t.items()}

    def restore_state(self, state):
        for k in TRI_KEYS:
            self._t[k].copy_(state[k])
        self.bump_version()

    # -- device methods (the reference's method boundary, csrc/bd_ops.cuh) --
    # Each runs one cooperative launch on this triangulation's device arrays
    # and the given positions (numpy or CUDA tensors), then returns host
    # values like the reference's numpy methods do.

    def _ops(self, n_pairs: int = 0):
        from ._ops import OpState
        self.bump_version()  # the op may rewrite the arrays: older host copies go stale
        return OpState(self.n_vertices, self.box.length, self.device, tri=self, n_pairs=n_pairs, tol=self.tol)

    def _pos(self, positions):
        import torch
        from ._ops import as_device
        return as_device(positions, torch.float64, self.device, (self.n_vertices, 2))

    def apply_crossings(self, crossings):
        """triangulation.py:166-177 (device)."""
        import torch
        from ._ops import as_device
        cr = as_device(crossings, torch.int64, self.device, (self.n_vertices, 2))
        op = self._ops()
        op.run("bd_tri_apply_crossings", ctypes.c_void_p(cr.data_ptr()))

    def signed_area2(self, positions) -> np.ndarray:
        """triangulation.py:186-191 (device): twice the signed area per triangle."""
        import torch
        out = torch.empty(self.n_triangles, dtype=torch.float64, device=self.device)
        op = self._ops().bind(pos=self._pos(positions))
        op.run("bd_tri_signed_area2", ctypes.c_void_p(out.data_ptr()))
        return out.cpu().numpy()

    def _edge_flags(self, name, positions, tol=None) -> np.ndarray:
        import torch
        out = torch.empty(self.n_edges, dtype=torch.uint8, device=self.device)
        op = self._ops().bind(pos=self._pos(positions))
        if tol is not None:
            op.p.tol = float(tol)
        op.run(name, ctypes.c_void_p(out.data_ptr()))
        return out.cpu().numpy().astype(bool)

    def delaunay_flags(self, positions, tol: float | None = None) -> np.ndarray:
        """triangulation.py:226-229 (device): right opposite vertex inside the left circumcircle."""
        return self._edge_flags("bd_tri_delaunay_flags", positions, tol)

    def inverted_edge_flags(self, positions) -> np.ndarray:
        """triangulation.py:231-234 (device): point-in-triangle inversion predicate."""
        return self._edge_flags("bd_tri_inverted_edge_flags", positions)

    def detect_inverted_triangles(self, positions) -> list:
        """triangulation.py:236-238"""
        flags = self.inverted_edge_flags(positions)
        return [FlipDecision(int(e), "inverted-triangle") for e in np.flatnonzero(flags)]

    def edge_inversion_present(self, prev, curr) -> bool:
        """triangulation.py:240-250 (device): some edge vector reversed its sign."""
        op = self._ops().bind(pos=self._pos(curr), prev=self._pos(prev))
        return bool(op.run("bd_tri_edge_inversion", op.res_ptr)[0])

    def flip_edge(self, e: int):
        """triangulation.py:254-302 (device): replace edge (a, b) by the cross diagonal (c, d)."""
        self.flip_edges([int(e)])

    def flip_edges(self, edges):
        """flip_edge for each edge in order (one launch)."""
        import torch
        ed = torch.as_tensor(np.asarray(edges, dtype=np.int64).reshape(-1)).to(self.device)
        op = self._ops()
        res = op.run("bd_tri_flip_edges", ctypes.c_void_p(ed.data_ptr()), int(ed.numel()), op.res_ptr)
        if res[0]:
            raise BrownsimError(f"edge {int(ed[int(res[1])])} cannot be flipped (degenerate or glued quad)")

    def restore_delaunay(self, positions, tol: float | None = None, max_passes: int = 1000) -> int:
        """triangulation.py:319-334 (device): Lawson flips in greedy
        ascending-edge independent sets until no in-circle violation; passes."""
        op = self._ops().bind(pos=self._pos(positions))
        if tol is not None:
            op.p.tol = float(tol)
        res = op.run("bd_tri_restore_delaunay_ex", int(max_passes), op.res_ptr)
        if res[0] == 2:
            raise NonConvergenceError(f"delaunay restoration did not converge in {max_passes} passes")
        if res[0]:
            raise BrownsimError(f"restore_delaunay: edge {int(res[1])} cannot be flipped")
        return int(res[1])

    def repair_inversions(self, positions, prev=None, max_passes: int = 10) -> RepairResult:
        """triangulation.py:336-363 (device): flip away inverted triangles;
        with `prev`, edges crossed by a vertex's path are flagged too."""
        pos = self._pos(positions)
        op = self._ops().bind(pos=pos, prev=self._pos(prev) if prev is not None else pos)
        res = op.run("bd_tri_repair_inversions", int(max_passes), int(prev is not None), op.res_ptr)
        if res[0]:
            raise BrownsimError(f"repair_inversions: device status {int(res[0])}")
        return RepairResult(int(res[1]), int(res[2]), bool(res[3]))

    # -- host-side geometry (validation / read-out only) --------------------

    def tri_coords(self, positions) -> np.ndarray:
        pos = np.asarray(positions, dtype=np.float64)
        return pos[self.tri_v] + self.tri_shift.astype(np.float64) * self.box.length

    def edge_quads(self, positions):
        return host_edge_quads(self.arrays(), positions, self.box.length)

    def canonical_edge_keys(self) -> set:
        """triangulation.py:484-496"""
        return canonical_edge_keys(self.arrays())

    def audit(self, positions, tol: float | None = None) -> AuditReport:
        return audit_arrays(self.arrays(), self.n_vertices, positions, self.box, self.tol if tol is None else tol)


# ---------------------------------------------------------------------------
# host helpers on plain numpy arrays


def host_edge_quads(a: dict, positions, L):
    pos = np.asarray(positions, dtype=np.float64)
    tl = a["edge_tri"][:, 0]
    tr = a["edge_tri"][:, 1]
    ol = a["edge_opp"][:, 0].astype(np.int64)
    orr = a["edge_opp"][:, 1].astype(np.int64)
    a_sl, b_sl, a_sr = (ol + 1) % 3, (ol + 2) % 3, (orr + 2) % 3
    sh = a["tri_shift"].astype(np.float64)
    tv = a["tri_v"]

    def emb(tri, slot, extra=None):
        s = sh[tri, slot]
        if extra is not None:
            s = s + extra
        return pos[tv[tri, slot]] + s * L

    A = emb(tl, a_sl)
    B = emb(tl, b_sl)
    C = emb(tl, ol)
    D = emb(tr, orr, extra=sh[tl, a_sl] - sh[tr, a_sr])
    return A, B, C, D


def incircle(a, b, c, d, tol: float = DEFAULT_TOL):
    """Lifted in-circle test, triangulation.py:66-87 (host, vectorised)."""
    a, b, c, d = (np.asarray(v, dtype=np.float64) for v in (a, b, c, d))
    ax, ay = a[..., 0] - d[..., 0], a[..., 1] - d[..., 1]
    bx, by = b[..., 0] - d[..., 0], b[..., 1] - d[..., 1]
    cx, cy = c[..., 0] - d[..., 0], c[..., 1] - d[..., 1]
    a2 = ax * ax + ay * ay
    b2 = bx * bx + by * by
    c2 = cx * cx + cy * cy
    det = ax * (by * c2 - b2 * cy) - ay * (bx * c2 - b2 * cx) + a2 * (bx * cy - by * cx)
    s = np.maximum.reduce([np.abs(ax), np.abs(ay), np.abs(bx), np.abs(by), np.abs(cx), np.abs(cy)])
    s2 = s * s
    return det > tol * (s2 * s2)


def canonical_edge_keys(a: dict) -> set:
    sh = a["tri_shift"].astype(np.int64)
    tl = a["edge_tri"][:, 0]
    ol = a["edge_opp"][:, 0].astype(np.int64)
    off = sh[tl, (ol + 2) % 3] - sh[tl, (ol + 1) % 3]
    ev = a["edge_v"].astype(np.int64)
    keys = set()
    for e in range(ev.shape[0]):
        va, vb = int(ev[e, 0]), int(ev[e, 1])
        o = (int(off[e, 0]), int(off[e, 1]))
        keys.add(min((va, vb, o), (vb, va, (-o[0], -o[1]))))
    return keys


def audit_arrays(a: dict, n_vertices: int, positions, box: PeriodicBox, tol: float) -> AuditReport:
    """Structural + geometric health report (triangulation.py:386-482), vectorised."""
    msgs = []
    V, E, F = n_vertices, a["edge_v"].shape[0], a["tri_v"].shape[0]
    euler_ok = (E == 3 * V) and (F == 2 * V)
    if not euler_ok:
        msgs.append(f"euler counts off: V={V} E={E} F={F} (want E=3V, F=2V)")
    et, eo, ev, tv, te = a["edge_tri"].astype(np.int64), a["edge_opp"].astype(np.int64), \
        a["edge_v"].astype(np.int64), a["tri_v"].astype(np.int64), a["tri_edge"].astype(np.int64)
    sh = a["tri_shift"].astype(np.int64)
    in_range = (et >= 0).all() and (et < F).all() and (eo >= 0).all() and (eo < 3).all() \
        and (te >= 0).all() and (te < E).all() and (tv >= 0).all() and (tv < V).all()
    refs_ok = bool(in_range)
    if in_range and E:
        tl, tr, ol, orr = et[:, 0], et[:, 1], eo[:, 0], eo[:, 1]
        ok = (tl != tr) & (te[tl, ol] == np.arange(E)) & (te[tr, orr] == np.arange(E)) \
            & (tv[tl, (ol + 1) % 3] == ev[:, 0]) & (tv[tl, (ol + 2) % 3] == ev[:, 1]) \
            & (tv[tr, (orr + 1) % 3] == ev[:, 1]) & (tv[tr, (orr + 2) % 3] == ev[:, 0])
        d_a = sh[tl, (ol + 1) % 3] - sh[tr, (orr + 2) % 3]
        d_b = sh[tl, (ol + 2) % 3] - sh[tr, (orr + 1) % 3]
        shift_ok = (d_a == d_b).all(axis=1)
        if not ok.all():
            msgs.append(f"{int((~ok).sum())} edges with broken cross references")
        if not (shift_ok | ~ok).all():
            msgs.append("incompatible image shifts between triangles")
        good = ok & shift_ok
        refs_ok = bool(good.all())
        if refs_ok:
            seen = np.zeros((F, 3), dtype=bool)
            seen[tl, ol] = True
            seen[tr, orr] = True
            if not seen.all():
                refs_ok = False
                msgs.append("some triangle edge slots are not referenced by any edge")
    elif not in_range:
        msgs.append("index arrays out of range; geometric checks skipped")
    shifts_in_range = bool(np.all(a["tri_shift"][:, 0, :] == 0) and np.all(np.abs(a["tri_shift"]) <= 1))
    if not shifts_in_range:
        msgs.append("image shifts outside {-1,0,1} (embedding regime exceeded)")
    if in_range:
        pos = np.asarray(positions, dtype=np.float64)
        xy = pos[tv] + sh.astype(np.float64) * box.length
        e1 = xy[:, 1] - xy[:, 0]
        e2 = xy[:, 2] - xy[:, 0]
        area2 = e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]
        n_bad_area = int(np.count_nonzero(area2 <= 0.0))
        if n_bad_area:
            msgs.append(f"{n_bad_area} triangles with non-positive area")
        A, B, C, D = host_edge_quads(a, pos, box.length)
        n_circ = int(np.count_nonzero(incircle(A, B, C, D, tol)))
        if n_circ:
            msgs.append(f"{n_circ} edges violate the in-circle condition")
        s0 = np.linalg.norm(xy[:, 1] - xy[:, 0], axis=1)
        s1 = np.linalg.norm(xy[:, 2] - xy[:, 1], axis=1)
        s2 = np.linalg.norm(xy[:, 0] - xy[:, 2], axis=1)
        with np.errstate(divide="ignore", invalid="ignore"):
            circum = np.where(area2 > 0.0, s0 * s1 * s2 / np.where(area2 > 0.0, area2, 1.0), np.inf)
        max_circum = float(np.max(circum)) if F else 0.0
        min_area = float(area2.min() / 2.0) if F else 0.0
    else:
        n_bad_area, n_circ, max_circum, min_area = 0, 0, float("inf"), 0.0
    circum_ok = bool(max_circum < box.length / 2.0)
    return AuditReport(V, E, F, euler_ok, refs_ok, min_area, n_bad_area, n_circ, max_circum, circum_ok,
                       shifts_in_range, msgs)


# ---------------------------------------------------------------------------
# one-time construction (restatement of triangulation.py:514-648)


def _lex_argmin3(keys):
    """keys: list of 3 arrays (T, m); index of the lexicographically smallest per row."""
    best = np.zeros(keys[0].shape[0], dtype=np.int64)
    cur = keys[0].copy()
    for r in (1, 2):
        cand = keys[r]
        # lexicographic cand < cur
        less = np.zeros(cand.shape[0], dtype=bool)
        eq = np.ones(cand.shape[0], dtype=bool)
        for j in range(cand.shape[1]):
            less |= eq & (cand[:, j] < cur[:, j])
            eq &= cand[:, j] == cur[:, j]
        best = np.where(less, r, best)
        cur = np.where(less[:, None], cand, cur)
    return best, cur


def _first_occurrence_order(rows: np.ndarray):
    """Unique rows in order of first occurrence: (inverse ids, first index per id)."""
    _, first, inv = np.unique(rows, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    return rank[inv.reshape(-1)], first[order]


def build_from_tiling(pos: np.ndarray, L: float, n: int, margin: int):
    """Arrays of _build_from_tiling (triangulation.py:553-648) or None."""
    from scipy.spatial import Delaunay as _PlanarDelaunay

    shifts = [(0, 0)] + [(sx, sy) for sy in range(-margin, margin + 1) for sx in range(-margin, margin + 1)
                         if (sx, sy) != (0, 0)]
    shift_arr = np.array(shifts, dtype=np.int64)
    cloud = np.concatenate([pos + shift_arr[c] * L for c in range(len(shifts))], axis=0)
    simp = _PlanarDelaunay(cloud).simplices.astype(np.int64)
    p0 = cloud[simp[:, 0]]
    e1 = cloud[simp[:, 1]] - p0
    e2 = cloud[simp[:, 2]] - p0
    cw = (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]) < 0
    simp[cw] = simp[cw][:, [0, 2, 1]]
    base = simp % n
    copy = simp // n
    fd = np.flatnonzero(np.any(copy == 0, axis=1))
    b = base[fd]
    s = shift_arr[copy[fd]]  # (T,3,2)
    # canonical rotation key: (b rotated, rel shifts of slots 1,2 w.r.t. slot 0)
    keys = []
    for r in range(3):
        idx = [(r + j) % 3 for j in range(3)]
        rb = b[:, idx]
        rs = s[:, idx, :]
        rel = np.concatenate([rs[:, 1] - rs[:, 0], rs[:, 2] - rs[:, 0]], axis=1)
        keys.append(np.concatenate([rb, rel], axis=1))
    _, kmin = _lex_argmin3(keys)
    tid, first = _first_occurrence_order(kmin)
    if first.size != 2 * n:
        return None
    # stored anchored at the first fundamental-domain slot
    fb, fs, fc = b[first], s[first], copy[fd][first]
    anchor = np.argmax(fc == 0, axis=1)
    idx = (anchor[:, None] + np.arange(3)[None, :]) % 3
    rb = np.take_along_axis(fb, idx, axis=1)
    rs = np.take_along_axis(fs, idx[:, :, None], axis=1)
    rs = rs - rs[:, 0:1, :]
    if np.any(np.abs(rs) > 1):
        return None
    tri_v = rb.astype(np.int32)
    tri_shift = rs.astype(np.int8)
    # edges in order of first appearance over (t, k)
    sl = tri_shift.astype(np.int64)
    T = 2 * n
    k = np.arange(3)
    u_sl, v_sl = (k + 1) % 3, (k + 2) % 3
    u = tri_v[:, u_sl].astype(np.int64)
    v = tri_v[:, v_sl].astype(np.int64)
    off = sl[:, v_sl, :] - sl[:, u_sl, :]  # (T,3,2)
    fwd = np.stack([u, v, off[..., 0], off[..., 1]], axis=-1).reshape(-1, 4)
    rev = np.stack([v, u, -off[..., 0], -off[..., 1]], axis=-1).reshape(-1, 4)
    le = np.ones(fwd.shape[0], dtype=bool)
    eq = np.ones(fwd.shape[0], dtype=bool)
    lt = np.zeros(fwd.shape[0], dtype=bool)
    for j in range(4):
        lt |= eq & (fwd[:, j] < rev[:, j])
        eq &= fwd[:, j] == rev[:, j]
    le = lt | eq
    key = np.where(le[:, None], fwd, rev)
    side = np.where(le, 0, 1)
    eid, efirst = _first_occurrence_order(key)
    if efirst.size != 3 * n:
        return None
    slot = eid * 2 + side
    if np.unique(slot).size != slot.size:
        return None  # two (t,k) claim the same side: inconsistent quotient
    if slot.size != 6 * n:
        return None
    edge_v = key[efirst][:, :2].astype(np.int32)
    edge_tri = np.empty((3 * n, 2), dtype=np.int32)
    edge_opp = np.empty((3 * n, 2), dtype=np.int8)
    tk_t = np.repeat(np.arange(T), 3)
    tk_k = np.tile(np.arange(3), T)
    edge_tri[eid, side] = tk_t
    edge_opp[eid, side] = tk_k
    tri_edge = eid.reshape(T, 3).astype(np.int32)
    return dict(tri_v=tri_v, tri_shift=tri_shift, tri_edge=tri_edge, edge_v=edge_v, edge_tri=edge_tri,
                edge_opp=edge_opp)


def build_initial_arrays(positions, box: PeriodicBox, tol: float = DEFAULT_TOL, restore=None):
    """Reference build_initial (triangulation.py:514-550) up to the final
    restore_delaunay/audit, which `restore(arrays) -> (arrays, report)` performs
    (on the GPU in build_initial)."""
    pos = np.asarray(positions, dtype=np.float64)
    n = pos.shape[0]
    if n < 3:
        raise BuildError(f"need at least 3 points to triangulate, got {n}")
    if np.unique(pos, axis=0).shape[0] != n:
        raise BuildError("coincident points cannot be triangulated")
    jittered = pos + build_jitter(n, box)
    last = ["no tiling produced a consistent quotient"]
    for margin in (1, 2, 3):
        arrays = build_from_tiling(jittered, box.length, n, margin)
        if arrays is None:
            continue
        if restore is None:
            return arrays
        arrays, report = restore(arrays)
        if report.euler_ok and report.refs_ok and report.n_nonpositive_areas == 0 \
                and report.n_incircle_violations == 0:
            return arrays
        last = report.messages
    raise BuildError("could not build a valid periodic triangulation; the point set is too sparse or too "
                     "degenerate for this box: " + "; ".join(last))


def build_jitter(n: int, box: PeriodicBox) -> np.ndarray:
    """The reference's build jitter (triangulation.py:536-540): 1e-9 L normals, fixed Philox key."""
    gen = np.random.Generator(np.random.Philox(key=np.array(_JITTER_KEY, dtype=np.uint64)))
    return gen.standard_normal((n, 2)) * (1e-9 * box.length)


BUILD_REASONS = {1: "coincident points", 2: "Voronoi cell polygon overflow",
                 3: "point set too sparse for the box (Voronoi cell not closed within half the box)",
                 4: "Delaunay degree above 32", 5: "neighbour image beyond the adjacent box copy",
                 6: "asymmetric neighbour relation (degenerate input)",
                 7: "inconsistent triangle (degenerate input)",
                 8: "repeated vertex in a triangle (too few points for the box)", 9: "Euler counts off"}


def device_build_tensors(jittered, box: PeriodicBox, device=None) -> dict:
    """The six arrays of the periodic Delaunay triangulation of `jittered`
    (n,2), built on the GPU (bd_tri_build_initial, csrc/bd_build.cuh), as
    device tensors.  Raises BuildError when the build fails."""
    import torch
    from ._lib import check, lib, require_cuda
    from .dynamics import _stream, _tri_struct
    require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    pts = np.ascontiguousarray(jittered, dtype=np.float64)
    n = pts.shape[0]
    if n < 3:
        raise BuildError(f"need at least 3 points to triangulate, got {n}")
    L = float(box.length)
    t = {k: torch.empty((m * n,) + _SHAPES[k], dtype=getattr(torch, np.dtype(_DTYPES[k]).name), device=dev)
         for k, m in (("tri_v", 2), ("tri_shift", 2), ("tri_edge", 2), ("edge_v", 3), ("edge_tri", 3),
                      ("edge_opp", 3))}
    pos_t = torch.from_numpy(pts).to(dev)
    wb = int(lib().bd_tri_build_workspace_bytes(n, L))
    work = torch.empty(wb // 8 + 64, dtype=torch.int64, device=dev)
    res = torch.zeros(4, dtype=torch.int64, device=dev)
    ts = _tri_struct(t, n)
    check(lib().bd_tri_build_initial(ctypes.c_void_p(pos_t.data_ptr()), n, L, ctypes.byref(ts),
                                     ctypes.c_void_p(work.data_ptr()), work.numel() * 8,
                                     ctypes.c_void_p(res.data_ptr()), _stream()), "bd_tri_build_initial")
    status, vertex, reason, _ = (int(v) for v in res.cpu().numpy())
    if status:
        raise BuildError(f"device triangulation build failed at vertex {vertex}: "
                         f"{BUILD_REASONS.get(reason, reason)}")
    return t


def build_initial(positions, box: PeriodicBox, tol: float = DEFAULT_TOL, device=None,
                  method: str = "host") -> PeriodicTriangulation:
    """Periodic Delaunay triangulation of wrapped positions; the clean-up
    flip pass (restore_delaunay) runs on the GPU.

    method="host": the reference's construction (Qhull on the jittered
    tiling), array for array identical to the reference's -- trajectories
    then match the reference bit for bit.  method="device": the whole build
    on the GPU (csrc/bd_build.cuh, ~1000x faster, and it also succeeds where
    the tiling fails); the same edge set as the reference's except where
    Qhull mis-decides an exactly cocircular quad of the unjittered points
    (both diagonals are Delaunay there), indexed by owner vertex."""
    from .dynamics import device_restore_delaunay

    pos = np.asarray(positions, dtype=np.float64)
    if method == "device":
        return build_initial_device(pos, box, tol, device)
    if method != "host":
        raise ValueError(f"unknown build method {method!r}")

    def restore(arrays):
        tri = PeriodicTriangulation(box, pos.shape[0], **arrays, tol=tol, device=device)
        device_restore_delaunay(tri, pos, box, tol)
        out = tri.arrays()
        return out, audit_arrays(out, pos.shape[0], pos, box, tol)

    arrays = build_initial_arrays(pos, box, tol, restore)
    return PeriodicTriangulation(box, pos.shape[0], **arrays, tol=tol, device=device)


def build_initial_device(positions, box: PeriodicBox, tol: float = DEFAULT_TOL, device=None) -> PeriodicTriangulation:
    """build_initial(method="device"): the reference's jitter, the device
    Voronoi/Delaunay build, restore_delaunay on the unjittered points and
    the geometric audit, all on the GPU (triangulation.py:514-550)."""
    import torch
    from ._lib import check, lib
    from .dynamics import _stream, _tri_struct, device_restore_delaunay, make_params
    from .core import SimParams
    pos = np.asarray(positions, dtype=np.float64)
    n = pos.shape[0]
    if n >= 3 and np.unique(pos, axis=0).shape[0] != n:
        raise BuildError("coincident points cannot be triangulated")
    t = device_build_tensors(pos + build_jitter(n, box), box, device)
    tri = PeriodicTriangulation(box, n, **t, tol=tol, device=device)
    device_restore_delaunay(tri, pos, box, tol)
    dev = tri.device
    pos_t = torch.from_numpy(np.ascontiguousarray(pos)).to(dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    from ._abi import BdState
    s = BdState()
    s.pos = pos_t.data_ptr()
    s.tri = _tri_struct(tri.tensors(), n)
    bp = make_params(SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.0), box.length, 0, 0)
    bp.tol = float(tol)
    check(lib().bd_tri_audit_geometry(ctypes.byref(s), ctypes.byref(bp), ctypes.c_void_p(out.data_ptr()),
                                      _stream()), "bd_tri_audit_geometry")
    bad_area, bad_circle = (int(v) for v in out.cpu().numpy())
    if bad_area or bad_circle:
        raise BuildError(f"device build failed the audit: {bad_area} non-positive areas, "
                         f"{bad_circle} in-circle violations")
    return tri
