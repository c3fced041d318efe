"""Golden files for the snapshot / per-step CSV formats (cli.py:263-321,
metrics.py:13-109), written by the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_io.py

Output: tests/golden/io/{inputs.npz, snapshot.txt, run.csv, run_short.csv,
flags.txt}: the inputs and the reference's files, compared byte for byte by
tests/test_io.py.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from brownsim.cli import write_locality_flags, write_snapshot  # noqa: E402
from brownsim.core import ParticleSystem, PeriodicBox  # noqa: E402
from brownsim.dynamics import StepStats  # noqa: E402
from brownsim.metrics import RunReport, write_csv  # noqa: E402

OUT = os.path.join(HERE, "io")


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(11)
    n, L = 257, 31.62277660168379
    pos = rng.uniform(0.0, L, size=(n, 2))
    pos[0] = (0.0, 0.1)            # exact zero, a non-representable decimal
    pos[1] = (5e-324, 1e-300)      # denormal, tiny
    pos[2] = (np.nextafter(L, 0.0), L / 3.0)
    types = rng.integers(0, 3, n).astype(np.int32)
    box = PeriodicBox(L)
    sys_ = ParticleSystem(pos.copy(), types, np.ones(n), np.ones(n), box)
    t = 12.345678901234567
    write_snapshot(sys_, t, os.path.join(OUT, "snapshot.txt"))
    flags = rng.random(n) < 0.2
    write_locality_flags(flags, os.path.join(OUT, "flags.txt"))
    rows = []
    for k in range(14):
        rows.append(dict(step=k, dt_used=0.01 * 0.5 ** (k % 3), overlap_iterations=int(rng.integers(0, 30)),
                         flip_passes=int(rng.integers(0, 9)), inversion_repairs=int(rng.integers(0, 3)),
                         rollbacks=k % 3, force_ms=float(rng.uniform(0, 50)), maintain_ms=float(rng.uniform(0, 5)),
                         overlap_ms=float(rng.uniform(0, 5)), step_ms=float(rng.uniform(50, 60))))
    cols = list(rows[0])
    np.savez(os.path.join(OUT, "inputs.npz"), pos=sys_.positions, types=types, L=L, t=t, flags=flags,
             series=np.array([[r[c] for c in cols] for r in rows], dtype=np.float64), cols=np.array(cols))
    write_csv(RunReport("cfg-test", n, [StepStats(**r) for r in rows], warmup=10), os.path.join(OUT, "run.csv"))
    # warmup >= series length: no summary rows (metrics.py:85)
    write_csv(RunReport("short", n, [StepStats(**r) for r in rows[:5]], warmup=10),
              os.path.join(OUT, "run_short.csv"))
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
