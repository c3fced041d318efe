"""compute-sanitizer over the flip / overlap kernels and the FAST-SYM pair
kernel (the reference's safety net is its determinism
contract, _kernels.py:1-9, tests/test_acceptance.py:287-313; the device
path adds race and memory checking).

  racecheck -- shared-memory hazards: the single-CTA shared-memory step
               driver (triangulation + scratch in smem) and the FAST-SYM
               kernel (TMA-filled tiles, mbarriers, per-warp sums)
  memcheck  -- out-of-bounds / misaligned accesses in every step kernel,
               the grid driver and the method-boundary ops
  synccheck -- illegal barrier usage (divergent __syncthreads / grid syncs)
Each run must report no hazard / error (racecheck: "0 hazards displayed
(0 errors, 0 warnings)", the others: "ERROR SUMMARY: 0 errors") and the workload's own
parity check must still pass (tools/sanitize_run.py prints OK)."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

CASES = [("racecheck", "smem", {}), ("racecheck", "sym", {}),
         ("memcheck", "smem", {}), ("memcheck", "grid", {"BD_BLOCK_MAX_N": "0"}), ("memcheck", "sym", {}),
         ("memcheck", "ops", {}), ("synccheck", "smem", {}), ("synccheck", "grid", {"BD_BLOCK_MAX_N": "0"})]


@pytest.mark.parametrize("tool,what,env", CASES, ids=[f"{t}-{w}" for t, w, _ in CASES])
def test_compute_sanitizer_clean(tool, what, env):
    if not os.path.exists(CS):
        pytest.skip("compute-sanitizer not installed")
    cmd = [CS, "--tool", tool, "--error-exitcode", "97"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), what]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, env={**os.environ, **env})
    out = r.stdout + r.stderr
    clean = "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck" \
        else "ERROR SUMMARY: 0 errors"
    assert clean in out and r.returncode == 0, out[-4000:]
    assert f"OK {what}" in out, out[-4000:]
