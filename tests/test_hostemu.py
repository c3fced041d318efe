"""The product's device step driver (csrc/bd_step.cuh, csrc/bd_allpairs.cuh)
compiled for the HOST with the ExecHost policy (tests/hostemu) -- checks the
driver's control flow and arithmetic on CPU: LFMIS flip selection, ordered
incidence gathers, rollback, crossings bookkeeping, exact min-image
breakpoints and the all-pairs image selector.  Test infrastructure only."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from golden_io import SCENARIOS, init_tri, load, pos_hash, tri_hash
from helpers import stats_row
from oracle import oracle as O
from paper_1703_02484_b200._abi import BdParams, BdState, BdStats, BdTri, c_d, c_i64, c_vp

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "hostemu", "_build", "libbd_hostemu.so")
TRI_KEYS = ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")


_LIB = None


def load_emu():
    """Build (make) and load the host-emulation library with its prototypes."""
    global _LIB
    if _LIB is not None:
        return _LIB
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "hostemu")], check=True, capture_output=True)
    lib = ctypes.CDLL(LIB)
    P = ctypes.POINTER
    lib.bdh_prepare_params.argtypes = [P(BdParams)]
    lib.bdh_workspace_bytes.argtypes = [P(BdParams), c_i64, c_i64]
    lib.bdh_workspace_bytes.restype = c_i64
    lib.bdh_step_tri.argtypes = [P(BdState), P(BdParams), P(BdStats)]
    lib.bdh_step_verlet.argtypes = [P(BdState), P(BdParams), P(BdStats)]
    lib.bdh_verlet_build.argtypes = [P(BdState), P(BdParams), c_d]
    lib.bdh_verlet_build.restype = c_i64
    lib.bdh_mi_fast.argtypes = [c_d, P(BdParams)]
    lib.bdh_mi_fast.restype = c_d
    lib.bdh_mi_ref.argtypes = [c_d, c_d]
    lib.bdh_mi_ref.restype = c_d
    lib.bdh_long_range_selector.argtypes = [c_vp, c_vp, c_vp, c_i64, P(BdParams), c_vp, c_vp]
    lib.bdh_normals.argtypes = [ctypes.c_uint64] * 4 + [c_i64, c_vp]
    lib.bdh_restore_delaunay.argtypes = [P(BdState), P(BdParams)]
    lib.bdh_restore_delaunay.restype = c_i64
    lib.bdh_step_abp.argtypes = [P(BdState), P(BdParams), P(BdStats)]
    lib.bdh_axis_select.argtypes = [c_d, c_d, c_d, c_d, c_vp, c_vp, c_vp]
    _LIB = lib
    return lib


@pytest.fixture(scope="module")
def emu():
    return load_emu()


def params_for(lib, L, seed=0, dt=0.01, r_cut=2.5, n=0, force_mode=0, pairs=False):
    from paper_1703_02484_b200.forces import verlet_pair_capacity
    p = BdParams()
    p.n = n
    p.L, p.sigma, p.dt, p.diffusion, p.cap, p.clamp = L, 1.0, dt, 0.01, 0.25, 3.0
    p.r_cut, p.skin, p.tol = r_cut, 0.5, 1e-12
    p.max_overlap_iters, p.max_rollbacks = 1000, 10
    p.seed, p.stream = seed, 2
    p.force_mode = force_mode
    lib.bdh_prepare_params(ctypes.byref(p))
    p.pair_capacity = verlet_pair_capacity(n, L, p.r_list) if pairs else 0
    return p


class HostState:
    """numpy-backed bd_state_t for the host driver."""

    def __init__(self, lib, rec, p):
        n = int(rec["n"])
        self.n = n
        self.pos = rec["pos0"].copy()
        self.prev = self.pos.copy()
        self.force = np.zeros_like(self.pos)
        self.alpha = rec["alpha"].copy()
        self.mu = rec["mu"].copy()
        self.ferr = np.zeros(n, np.int64)
        self.image = np.zeros((n, 2), np.int32)
        self.flags = np.zeros(n, np.uint8)
        has_tri = "init_tri_v" in rec
        self.tri = {k: v.copy() for k, v in init_tri(rec).items()} if has_tri else None
        self.bk = {k: v.copy() for k, v in self.tri.items()} if has_tri else None
        self.call = np.zeros(1, np.uint64)
        cap = max(int(p.pair_capacity), 1)
        self.pa = np.zeros(cap, np.int64)
        self.pb = np.zeros(cap, np.int64)
        self.snap = np.zeros((n, 2))
        self.meta = np.zeros(8, np.int64)
        ne = self.tri["edge_v"].shape[0] if has_tri else 0
        nt = self.tri["tri_v"].shape[0] if has_tri else 0
        self.work = np.zeros(lib.bdh_workspace_bytes(ctypes.byref(p), ne, nt) // 8 + 64, np.float64)
        ts = lambda a: BdTri(n, a["edge_v"].shape[0], a["tri_v"].shape[0], *[a[k].ctypes.data for k in TRI_KEYS])
        self.s = BdState(self.pos.ctypes.data, self.prev.ctypes.data, self.force.ctypes.data,
                         self.alpha.ctypes.data, self.mu.ctypes.data, self.ferr.ctypes.data,
                         self.image.ctypes.data, self.flags.ctypes.data, ts(self.tri) if has_tri else BdTri(),
                         ts(self.bk) if has_tri else BdTri(), self.call.ctypes.data, 0, self.pa.ctypes.data,
                         self.pb.ctypes.data, self.snap.ctypes.data, self.meta.ctypes.data, self.work.ctypes.data,
                         self.work.nbytes)


@pytest.mark.parametrize("worklist", [False, True], ids=["full-passes", "worklist"])
@pytest.mark.parametrize("name", SCENARIOS)
def test_host_driver_matches_reference(emu, name, worklist, monkeypatch):
    """Both restore_delaunay variants (every pass re-flags all edges / later
    passes re-flag only the worklist; chosen by edge count, forced here)."""
    if worklist:
        monkeypatch.setenv("BD_WORKLIST_MIN_EDGES", "0")
    rec = load(name)
    fm = int(rec["force_mode"])
    verlet = str(rec["mode"]) == "verlet"
    p = params_for(emu, float(rec["L"]), int(rec["seed"]), float(rec["dt"]), float(rec["r_cutoff"]),
                   n=int(rec["n"]), force_mode=1 if verlet else fm, pairs=verlet or fm != 0)
    h = HostState(emu, rec, p)
    st = BdStats()
    for s in range(len(rec["pos_hash"])):
        if verlet:
            emu.bdh_step_verlet(ctypes.byref(h.s), ctypes.byref(p), ctypes.byref(st))
        else:
            emu.bdh_step_tri(ctypes.byref(h.s), ctypes.byref(p), ctypes.byref(st))
        assert st.status == 0
        assert stats_row(st) == list(rec["stats"][s]), f"step {s}"
        assert pos_hash(h.pos) == rec["pos_hash"][s], f"step {s}"
        if h.tri is not None:
            assert tri_hash(h.tri) == rec["tri_hash"][s], f"step {s}"
    assert int(h.call[0]) == int(rec["calls"][-1])
    if "rebuilds" in rec:
        assert int(h.meta[2]) == int(rec["rebuilds"])


def test_host_verlet_pairs_match_reference_order(emu):
    k = load("kernels")
    pos, L = k["sr_pos"], float(k["sr_L"])
    n = pos.shape[0]
    rec = {"n": n, "pos0": pos, "alpha": np.zeros(n), "mu": np.zeros(n)}
    p = params_for(emu, L, n=n, r_cut=2.5, pairs=True)
    h = HostState(emu, rec, p)
    m = emu.bdh_verlet_build(ctypes.byref(h.s), ctypes.byref(p), 1.5)
    assert m == k["sr_pa"].size
    assert np.array_equal(h.pa[:m], k["sr_pa"]) and np.array_equal(h.pb[:m], k["sr_pb"])
    assert int(h.meta[3]) == k["sr_oa"].size


def test_host_brute_verlet_order(emu):
    k = load("kernels")
    pos, L = k["bf_pos"], float(k["bf_L"])
    n = pos.shape[0]
    rec = {"n": n, "pos0": pos, "alpha": np.zeros(n), "mu": np.zeros(n)}
    p = params_for(emu, L, n=n, r_cut=2.5, pairs=True)
    assert p.ncx == 0
    h = HostState(emu, rec, p)
    m = emu.bdh_verlet_build(ctypes.byref(h.s), ctypes.byref(p), 0.0)
    assert np.array_equal(h.pa[:m], k["bf_pa"]) and np.array_equal(h.pb[:m], k["bf_pb"])


@pytest.mark.parametrize("L", [25.888345500742656, 31.0, 585.7893, 1171.5729, 414.2135623730951, 3.0])
def test_min_image_breakpoints_exact(emu, L):
    p = params_for(emu, L)
    rng = np.random.default_rng(7)
    ds = list(rng.uniform(-L, L, 5000))
    for base in (p.mi_hi, p.mi_lo, L / 2, -L / 2):
        x = base
        for _ in range(4):
            ds += [x]
            x = np.nextafter(x, np.inf)
        x = base
        for _ in range(4):
            x = np.nextafter(x, -np.inf)
            ds += [x]
    for d in ds:
        d = float(d)
        if -L < d < L:
            assert emu.bdh_mi_fast(d, ctypes.byref(p)) == emu.bdh_mi_ref(d, L), d


@pytest.mark.parametrize("L", [25.888345500742656, 17.0, 585.7893, 1171.5729, 3.0])
def test_axis_select_breakpoint_is_the_bisection_result(emu, L):
    """axis_select walks from s = x - thr to the breakpoint; it must return
    exactly what a bisection over the bit patterns of [0, L) returns."""
    p = params_for(emu, L)
    smax = int(np.float64(L).view(np.uint64)) - 1
    bits = lambda b: float(np.uint64(b).view(np.float64))
    rng = np.random.default_rng(3)
    xs = list(rng.uniform(0, L, 400)) + [0.0, np.nextafter(0, 1), L / 2, np.nextafter(L / 2, 0),
                                         np.nextafter(L / 2, L), np.nextafter(L, 0), p.mi_hi, -p.mi_lo]
    T, sh, amb = ctypes.c_uint64(), (ctypes.c_double * 2)(), ctypes.c_int()
    for x in xs:
        x = float(x)
        emu.bdh_axis_select(x, L, p.mi_lo, p.mi_hi, ctypes.byref(T), sh, ctypes.byref(amb))
        up, down = (x - 0.0) >= p.mi_hi, (x - bits(smax)) < p.mi_lo
        if amb.value or not (up or down):
            assert T.value == (1 << 64) - 1
            continue
        thr = p.mi_hi if up else p.mi_lo
        good, bad = 0, smax + 1
        if x - bits(smax) >= thr:
            good = smax
        else:
            while bad - good > 1:
                mid = (good + bad) // 2
                if x - bits(mid) >= thr:
                    good = mid
                else:
                    bad = mid
        assert T.value == good, x


@pytest.mark.parametrize("L", [25.888345500742656, 17.0, 585.7893, 414.2135623730951])
def test_all_pairs_image_selector_bitwise(emu, L):
    p = params_for(emu, L)
    rng = np.random.default_rng(1)
    n = 400
    pos = rng.uniform(0, L, (n, 2))
    special = [0.0, L / 2, np.nextafter(L / 2, 0), np.nextafter(L / 2, L), p.mi_hi, np.nextafter(p.mi_hi, 0),
               -p.mi_lo, np.nextafter(L, 0), np.nextafter(0, 1)]
    for j, s in enumerate(special):
        pos[j, 0] = s
        pos[j + 20, 1] = s
        pos[j + 40] = [s, special[-1 - j]]
    pos[100] = [1.0, 2.0]
    pos[101] = [1.0 + L / 2, 2.0]
    pos[102] = [1.0, 2.0 + L / 2]
    pos = np.mod(pos, L)
    a = rng.normal(size=n)
    m = rng.normal(size=n)
    ref, rerr = O.long_range(pos, a, m, L)
    out = np.empty((n, 2))
    err = np.empty(n, np.int64)
    emu.bdh_long_range_selector(pos.ctypes.data, a.ctypes.data, m.ctypes.data, n, ctypes.byref(p), out.ctypes.data,
                                err.ctypes.data)
    assert np.array_equal(out, ref) and np.array_equal(err, rerr)


def test_device_noise_source_matches_numpy(emu):
    from oracle.noise_np import normal_pairs
    out = np.empty((5000, 2))
    emu.bdh_normals(9, 2, 4, 0, 5000, out.ctypes.data)
    assert np.array_equal(out, normal_pairs(9, 2, 4, 5000))


def test_host_restore_delaunay_matches_reference_build(emu):
    b = load("build")
    for tag in ("a", "b"):
        pos, L = b[f"{tag}_pos"], float(b[f"{tag}_L"])
        rec = {"n": pos.shape[0], "pos0": pos, "alpha": np.zeros(pos.shape[0]), "mu": np.zeros(pos.shape[0])}
        for k in TRI_KEYS:
            rec["init_" + k] = b[f"{tag}_pre_{k}"]
        p = params_for(emu, L, n=pos.shape[0])
        h = HostState(emu, rec, p)
        assert emu.bdh_restore_delaunay(ctypes.byref(h.s), ctypes.byref(p)) >= 0
        for k in TRI_KEYS:
            assert np.array_equal(h.tri[k], b[f"{tag}_fin_{k}"]), (tag, k)


@pytest.mark.parametrize("case", ["singular", "nonfinite"])
def test_host_step_error_paths(emu, case):
    """The fused check phase of the step driver (singularity, then
    finiteness, with the rollback backup in the same phase): the status
    and the offending indices of forces.py:54-58 / dynamics.py:84-86, and
    an untouched state."""
    from paper_1703_02484_b200._abi import BD_ERR_SINGULAR, BD_ERR_STEPFAIL
    rec = load("lr_c0_n256")
    p = params_for(emu, float(rec["L"]), int(rec["seed"]), float(rec["dt"]), float(rec["r_cutoff"]),
                   n=int(rec["n"]), force_mode=0)
    h = HostState(emu, rec, p)
    if case == "singular":
        h.pos[20] = h.pos[10]
    else:
        h.alpha[7] = np.nan
    pos0 = h.pos.copy()
    tri0 = {k: v.copy() for k, v in h.tri.items()}
    st = BdStats()
    emu.bdh_step_tri(ctypes.byref(h.s), ctypes.byref(p), ctypes.byref(st))
    if case == "singular":
        assert (st.status, st.err_i, st.err_k) == (BD_ERR_SINGULAR, 10, 20)
    else:
        assert st.status == BD_ERR_STEPFAIL and st.err_i == 0
    assert np.array_equal(h.pos, pos0)
    assert all(np.array_equal(h.tri[k], tri0[k]) for k in tri0)
