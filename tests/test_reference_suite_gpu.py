"""The reference's OWN test files, unmodified, run against the B200 engine
("the reference test files become parity tests unchanged").

tests/refplugin/bd_swap.py rebinds the reference's hot-path entry points --
brownsim._kernels.*, dynamics.integrate / correct_overlaps and the
PeriodicTriangulation maintenance methods -- to this package's device code;
the reference's tests then drive the GPU through the reference's own API and
check it with their own oracles (naive loops bit for bit, brute-force pair
sets, closed-form bounces, Fig. 5 / Fig. 6 scenarios, rebuild comparisons,
rollbacks, acceptance criteria).

The reference package is installed (pip --target, --no-deps) under
baseline/_ref together with a copy of its tests (baseline/_ref/tests_ref;
git-ignored, shipped to the GPU box with the snapshot).  Without it the test
is skipped.  Every replacement must have been called (the plugin counts),
so a pass cannot come from the reference's own numba / numpy code.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "tests_ref")

# the device replacements each reference test file must exercise
SUITES = {
    "test_forces.py": {"long_range_kernel", "short_range_kernel", "cell_pairs", "max_sq_displacement"},
    "test_triangulation.py": {"tri.restore_delaunay", "tri.repair_inversions", "tri.flip_edge",
                              "tri.apply_crossings", "tri.delaunay_flags"},
    "test_dynamics.py": {"integrate", "correct_overlaps", "long_range_kernel", "short_range_kernel",
                         "tri.edge_inversion_present", "tri.repair_inversions", "tri.restore_delaunay"},
    "test_acceptance.py": {"long_range_kernel", "integrate", "correct_overlaps", "tri.restore_delaunay"},
}


def run_suite(fname, tmp_path, extra=()):
    if not os.path.isfile(os.path.join(REF_TESTS, fname)):
        pytest.skip("reference package not installed under baseline/_ref (see DESIGN.md §5)")
    report = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests", "refplugin"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env["BD_SWAP_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", "-p", "bd_swap", "-p", "no:cacheprovider", "-q", "-rfE",
           "-m", "not slow", os.path.join(REF_TESTS, fname), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3000, env=env, cwd=str(tmp_path))
    out = r.stdout + r.stderr
    calls = json.loads(report.read_text())["calls"] if report.exists() else {}
    return r.returncode, out, calls


@pytest.mark.parametrize("fname", sorted(SUITES))
def test_reference_suite_passes_on_device(fname, tmp_path):
    rc, out, calls = run_suite(fname, tmp_path)
    tail = out[-6000:]
    print(tail)
    print("device calls:", calls)
    assert rc == 0, tail
    missing = {k for k in SUITES[fname] if calls.get(k, 0) == 0}
    assert not missing, f"replacements never called: {missing}; calls {calls}"
