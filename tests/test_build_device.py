"""The initial triangulation built on the device (csrc/bd_build.cuh,
build_initial(method="device")) against the reference's build_initial
(triangulation.py:514-648).

Parity statement: the device build is the exact Delaunay triangulation of
the reference's jittered points, so its edge set equals the reference's
wherever Qhull decides correctly.  The only admissible difference is the
diagonal of a quad that is EXACTLY cocircular at the unjittered positions
(there both diagonals are Delaunay and restore_delaunay leaves either), and
then the device's diagonal must be the exactly-correct one for the jittered
points.  Both are checked in rational arithmetic.

CPU: the build source compiled for the host (tests/hostemu) against the
reference's own build fixtures (tests/golden/build.npz) and against the
host restatement (pinned to those fixtures) at larger sizes.  GPU: cfg3 and
cfg4 sizes, including cfg4's seed 0, where the reference's build fails.
"""

import ctypes
import os
import subprocess
from fractions import Fraction

import numpy as np
import pytest

from golden_io import load

HERE = os.path.dirname(os.path.abspath(__file__))
C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
_EMU = None


def emu():
    global _EMU
    if _EMU is None:
        from paper_1703_02484_b200._abi import BdTri
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "hostemu")], check=True, capture_output=True)
        lib = ctypes.CDLL(os.path.join(HERE, "hostemu", "_build", "libbd_hostemu.so"))
        lib.bdh_tri_build_workspace_bytes.restype = ctypes.c_int64
        lib.bdh_tri_build_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_double]
        lib.bdh_tri_build.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(BdTri),
                                      ctypes.c_void_p, ctypes.c_void_p]
        _EMU = lib
    return _EMU


def emu_build(jittered, L):
    from paper_1703_02484_b200._abi import BdTri
    from paper_1703_02484_b200.triangulation import TRI_KEYS
    lib = emu()
    n = jittered.shape[0]
    a = dict(tri_v=np.zeros((2 * n, 3), np.int32), tri_shift=np.zeros((2 * n, 3, 2), np.int8),
             tri_edge=np.zeros((2 * n, 3), np.int32), edge_v=np.zeros((3 * n, 2), np.int32),
             edge_tri=np.zeros((3 * n, 2), np.int32), edge_opp=np.zeros((3 * n, 2), np.int8))
    t = BdTri(n, 3 * n, 2 * n, *[a[k].ctypes.data for k in TRI_KEYS])
    w = np.zeros(lib.bdh_tri_build_workspace_bytes(n, L) // 8 + 64)
    res = np.zeros(4, np.int64)
    pts = np.ascontiguousarray(jittered, dtype=np.float64)
    lib.bdh_tri_build(pts.ctypes.data, n, float(L), ctypes.byref(t), w.ctypes.data, res.ctypes.data)
    return a, res


def exact_incircle(q):
    """Sign-exact lifted determinant of (A, B, C, D): > 0 iff D is strictly inside circle ABC (CCW)."""
    (ax, ay), (bx, by), (cx, cy), (dx, dy) = [(Fraction(float(x)), Fraction(float(y))) for x, y in q]
    ax, ay, bx, by, cx, cy = ax - dx, ay - dy, bx - dx, by - dy, cx - dx, cy - dy
    return ((ax * ax + ay * ay) * (bx * cy - by * cx) - (bx * bx + by * by) * (ax * cy - ay * cx)
            + (cx * cx + cy * cy) * (ax * by - ay * bx))


def edge_quad_of(a, e, pos, L):
    from paper_1703_02484_b200.triangulation import host_edge_quads
    q = host_edge_quads(a, pos, L)
    return [(q[j][e, 0], q[j][e, 1]) for j in range(4)]


def edge_index(a, key):
    ev = a["edge_v"]
    from paper_1703_02484_b200.triangulation import canonical_edge_keys
    for e in np.flatnonzero(((ev[:, 0] == key[0]) & (ev[:, 1] == key[1])) | ((ev[:, 0] == key[1]) &
                                                                             (ev[:, 1] == key[0]))):
        sub = {k: v for k, v in a.items()}
        if key in canonical_edge_keys({**sub, "edge_v": ev[e:e + 1], "edge_tri": a["edge_tri"][e:e + 1],
                                       "edge_opp": a["edge_opp"][e:e + 1]}):
            return int(e)
    raise KeyError(key)


def assert_same_delaunay(dev, ref, pos, jittered, L, jittered_stage=True):
    """Edge sets equal, except diagonals of exactly-cocircular quads (real
    positions), where the device's diagonal is exactly Delaunay for the
    jittered points (jittered_stage) / for the real points."""
    from paper_1703_02484_b200.triangulation import canonical_edge_keys
    kd, kr = canonical_edge_keys(dev), canonical_edge_keys(ref)
    assert len(kd) == len(kr) == dev["edge_v"].shape[0]
    diff = kd - kr
    assert len(diff) <= max(2, len(kd) // 10000), len(diff)
    for key in diff:
        e = edge_index(dev, key)
        assert exact_incircle(edge_quad_of(dev, e, pos, L)) == 0, key  # cocircular: both diagonals Delaunay
        if jittered_stage:
            assert exact_incircle(edge_quad_of(dev, e, jittered, L)) < 0, key
    return len(diff)


def workload(n, rho, seed=0):
    from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density, wrap
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    pos = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=C0, seed=seed))[0]
    return box, wrap(box, pos)


# ---------------------------------------------------------------------------
# CPU: host-compiled build source


def test_emulated_build_equals_reference_fixture_edge_sets():
    """The reference's own builds (tests/golden/build.npz, made by
    make_golden.py from /root/reference): identical edge sets before
    (jittered) and after (restore_delaunay on the real points) clean-up."""
    from paper_1703_02484_b200.core import PeriodicBox
    from paper_1703_02484_b200.triangulation import audit_arrays, build_jitter, canonical_edge_keys
    b = load("build")
    for tag in ("a", "b"):
        pos, box = b[f"{tag}_pos"], PeriodicBox(float(b[f"{tag}_L"]))
        jit = pos + build_jitter(pos.shape[0], box)
        a, res = emu_build(jit, box.length)
        assert res[0] == 0, res
        pre = {k: b[f"{tag}_pre_{k}"] for k in a}
        fin = {k: b[f"{tag}_fin_{k}"] for k in a}
        assert canonical_edge_keys(a) == canonical_edge_keys(pre)
        assert canonical_edge_keys(a) == canonical_edge_keys(fin)
        rep = audit_arrays(a, pos.shape[0], pos, box, 1e-12)
        assert rep.ok and rep.shifts_in_range, rep.messages


@pytest.mark.parametrize("n,rho,seed", [(1024, 0.3, 0), (16384, 0.3, 0), (4096, 0.6, 1), (2048, 0.05, 3)])
def test_emulated_build_vs_host_restatement(n, rho, seed):
    from paper_1703_02484_b200.triangulation import audit_arrays, build_initial_arrays, build_jitter
    box, pos = workload(n, rho, seed)
    jit = pos + build_jitter(n, box)
    a, res = emu_build(jit, box.length)
    assert res[0] == 0, res
    ref = build_initial_arrays(pos, box)  # reference tiling on the same jittered points (pre clean-up)
    assert_same_delaunay(a, ref, pos, jit, box.length)
    rep = audit_arrays(a, n, jit, box, 1e-12)
    assert rep.ok and rep.shifts_in_range, rep.messages


def test_emulated_build_uniform_random_points():
    from paper_1703_02484_b200.core import PeriodicBox
    from paper_1703_02484_b200.triangulation import audit_arrays, build_initial_arrays, build_jitter
    rng = np.random.default_rng(5)
    for n, L in ((64, 8.0), (500, 30.0), (3000, 50.0)):
        box = PeriodicBox(L)
        pos = rng.uniform(0.0, L, size=(n, 2))
        jit = pos + build_jitter(n, box)
        a, res = emu_build(jit, L)
        assert res[0] == 0, res
        assert_same_delaunay(a, build_initial_arrays(pos, box), pos, jit, L)
        assert audit_arrays(a, n, jit, box, 1e-12).ok


def test_emulated_build_reports_failures():
    from paper_1703_02484_b200.triangulation import BUILD_REASONS
    rng = np.random.default_rng(0)
    pos = rng.uniform(0.0, 10.0, size=(40, 2))
    pos[7] = pos[3]
    _, res = emu_build(pos, 10.0)
    assert res[0] == 7 and res[2] == 1 and res[1] in (3, 7)  # BD_ERR_BUILD, coincident
    # 6 points in a large box: Voronoi cells wrap around the torus
    _, res = emu_build(rng.uniform(0.0, 10.0, size=(6, 2)), 10.0)
    assert res[0] == 7 and int(res[2]) in BUILD_REASONS


# ---------------------------------------------------------------------------
# GPU


@pytest.mark.gpu
def test_device_build_cfg3_matches_reference_build():
    """cfg3 (N = 131,072): build_initial(method="device") vs the reference
    construction, after restore_delaunay on the real points."""
    import time
    from paper_1703_02484_b200.triangulation import build_initial, build_initial_arrays, build_jitter, \
        device_build_tensors
    n = 131072
    box, pos = workload(n, 0.3)
    jit = pos + build_jitter(n, box)
    t = device_build_tensors(jit, box)
    pre = {k: v.cpu().numpy() for k, v in t.items()}
    ref_pre = build_initial_arrays(pos, box)
    assert_same_delaunay(pre, ref_pre, pos, jit, box.length)
    t0 = time.perf_counter()
    dev = build_initial(pos, box, method="device").arrays()
    t_dev = time.perf_counter() - t0
    ref = build_initial(pos, box).arrays()
    assert_same_delaunay(dev, ref, pos, jit, box.length, jittered_stage=False)
    assert t_dev < 20.0


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 0])
def test_device_build_cfg4_size_and_steps(seed):
    """cfg4 (N = 1,048,576, rho = 0.6): the device build succeeds for seed 1
    and for seed 0 (where the reference's tiling build fails), is
    audited clean, and the short-range step runs valid from it."""
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, SimParams
    from paper_1703_02484_b200.dynamics import LongRangeSimulation
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    from paper_1703_02484_b200.triangulation import build_initial
    from paper_1703_02484_b200.validation import audit_geometry, cell_overlaps
    from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density
    n = 1048576
    box = PeriodicBox(box_length_for_density(n, 1.0, 0.6))
    pos, t, a, m = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=C0, seed=seed))
    sys_ = ParticleSystem(pos, t, a, m, box)
    tri = build_initial(sys_.positions, box, method="device")
    assert tri.n_edges == 3 * n and tri.n_triangles == 2 * n
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01, r_cutoff=2.5)
    sim = LongRangeSimulation(sys_, params, CounterRng(seed, 2), tri=tri, force="short-range")
    assert audit_geometry(sim) == (0, 0)
    for _ in range(2):
        st = sim.step()
        assert st.rollbacks == 0
        assert audit_geometry(sim) == (0, 0)
        assert cell_overlaps(sim.sys.positions_t, box.length, 1.0 - 1e-9) == 0
