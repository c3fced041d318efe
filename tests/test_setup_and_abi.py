"""Host-side setup restatements and the C-ABI library (no GPU needed).

* init_system / build_initial restatements produce the reference's exact
  arrays (golden fixtures from the reference);
* libbd_b200.so loads and exports every entry point include/bd_b200.h
  declares; the ctypes struct mirrors match the header layout."""

import ctypes
import os
import re

import numpy as np
import pytest

from golden_io import SCENARIOS, load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]


@pytest.mark.parametrize("name", SCENARIOS)
def test_init_arrays_equal_reference_initial_state(name):
    from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density, wrap
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    rec = load(name)
    n, rho, seed = int(rec["n"]), float(rec["rho"]), int(rec["seed"])
    types = C0 if not name.startswith("lr_c3") else [(0.5, 3.0, -3.0), (0.5, -3.0, 3.0)]
    if name.startswith("lr_rollback"):
        types = [(0.5, 3.0, 3.0), (0.5, -3.0, -3.0)]
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    assert box.length == float(rec["L"])
    pos, _, alpha, mu = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=types, seed=seed))
    assert np.array_equal(wrap(box, pos), rec["pos0"])
    assert np.array_equal(alpha, rec["alpha"]) and np.array_equal(mu, rec["mu"])


def test_build_quotient_arrays_equal_reference():
    from paper_1703_02484_b200.core import PeriodicBox
    from paper_1703_02484_b200.triangulation import build_initial_arrays
    b = load("build")
    for tag in ("a", "b"):
        arrays = build_initial_arrays(b[f"{tag}_pos"], PeriodicBox(float(b[f"{tag}_L"])))
        for k, v in arrays.items():
            assert np.array_equal(v, b[f"{tag}_pre_{k}"]), (tag, k)


def test_audit_of_reference_build_is_clean():
    from paper_1703_02484_b200.core import PeriodicBox
    from paper_1703_02484_b200.triangulation import audit_arrays
    b = load("build")
    for tag in ("a", "b"):
        a = {k: b[f"{tag}_fin_{k}"] for k in ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")}
        rep = audit_arrays(a, b[f"{tag}_pos"].shape[0], b[f"{tag}_pos"], PeriodicBox(float(b[f"{tag}_L"])), 1e-12)
        assert rep.ok and rep.shifts_in_range
        a["edge_tri"] = a["edge_tri"].copy()
        a["edge_tri"][4, 0] = (a["edge_tri"][4, 0] + 1) % a["tri_v"].shape[0]
        assert not audit_arrays(a, b[f"{tag}_pos"].shape[0], b[f"{tag}_pos"], PeriodicBox(float(b[f"{tag}_L"])),
                                1e-12).refs_ok


@pytest.fixture(scope="module")
def cuda_lib():
    from paper_1703_02484_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def header_functions():
    src = open(os.path.join(ROOT, "include", "bd_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(bd_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol(cuda_lib):
    from paper_1703_02484_b200 import _abi
    names = header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(cuda_lib, n)]
    assert not missing, missing
    assert set(names) <= set(_abi.EXPORTS) | {"bd_probe_fp64"}


def test_struct_layouts_match_header(cuda_lib):
    """ctypes mirrors agree with the compiled layout (sizes via the workspace helpers)."""
    from paper_1703_02484_b200 import _abi
    assert ctypes.sizeof(_abi.BdTri) == 3 * 8 + 6 * 8
    assert ctypes.sizeof(_abi.BdStats) == 40 * 8
    p = _abi.BdParams()
    p.L, p.sigma, p.skin, p.r_cut = 100.0, 1.0, 0.5, 2.5
    cuda_lib.bd_prepare_params.argtypes = [ctypes.POINTER(_abi.BdParams)]
    cuda_lib.bd_prepare_params(ctypes.byref(p))
    assert p.r_list == 3.0 and p.ncx == 33
    assert p.mi_hi <= 50.0 and p.mi_lo >= -50.0


def test_roofline_accounting_and_bench_imports():
    """The host-side byte accounting used by bench.py / run_configs.py, and
    that the measurement scripts import and parse their arguments on CPU."""
    import subprocess
    import sys
    from paper_1703_02484_b200 import _abi
    from paper_1703_02484_b200.roofline import hbm_peak_gbs, phase_breakdown, phase_roofline, step_bytes
    work = {k: 0 for k in _abi.WORK_KEYS}
    work.update(integrate=1, flag_pass=2, overlap_pass=3, t_maintain_ns=1000, t_overlap_ns=500, t_total_ns=2000)
    n, ne, nt = 1000, 3000, 2000
    assert step_bytes(work, n, ne, nt) == 64 * n + 2 * (11 * ne + 18 * nt + 16 * n) + 3 * (8 * ne + 32 * n)
    ph = phase_roofline(work, n, ne, nt)
    assert set(ph) == {"maintenance", "overlap"} and ph["overlap"]["GBs"] == 3 * (8 * ne + 32 * n) / 500
    assert abs(sum(phase_breakdown(work).values()) - 1.0) < 1e-12
    assert hbm_peak_gbs({"hbm_gbs": 6545.9}) == 6545.9 and hbm_peak_gbs({}) > 0
    for script in ("bench.py", "tools/run_configs.py"):
        r = subprocess.run([sys.executable, os.path.join(ROOT, script), "--help"], capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]


def test_stepstats_phase_timings_follow_the_reference_meaning():
    """StepStats force/maintain/overlap ms (dynamics.py:193-270, :328-341)
    from the step kernel's device timers: triangulation steps split
    maintenance from overlap rounds; Verlet steps report the list rebuild as
    maintain and the short-range force as force."""
    from paper_1703_02484_b200.dynamics import _phase_ms
    work = {"t_maintain_ns": 300_000, "t_overlap_ns": 250_000, "t_incidence_ns": 50_000, "t_sr_force_ns": 20_000,
            "t_verlet_ns": 40_000}
    f, m, o = _phase_ms(work, 9.5, 0.8, True)
    assert (round(f, 6), round(m, 6), round(o, 6)) == (9.52, 0.3, 0.3)
    f, m, o = _phase_ms(work, 0.0, 0.5, False)
    assert (round(f, 6), round(m, 6), round(o, 6)) == (0.02, 0.04, 0.44)
