"""Per-step device time of the O(N) step kernel (and the force) for the
config sizes, with the driver selected by the environment (BD_CLUSTER_*,
BD_BLOCK_MAX_N, BD_SMEM_DRIVER, ...).  Measurement only.
    python tools/time_step.py cfg1 cfg2 n4096 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
CFG = {"n256": (256, 0.3, "long-range", "exact", 0), "n512": (512, 0.3, "long-range", "exact", 0),
       "n1536": (1536, 0.3, "long-range", "exact", 0), "n32768": (32768, 0.3, "long-range", "fast-sym", 0),
       "n49152": (49152, 0.3, "long-range", "fast-sym", 0),
       "cfg1": (1024, 0.3, "long-range", "exact", 0), "cfg2": (16384, 0.3, "short-range", "exact", 0),
       "n4096": (4096, 0.3, "long-range", "exact", 0), "n8192": (8192, 0.3, "long-range", "fast-sym", 0),
       "cfg5": (65536, 0.3, "long+short", "fast-sym", 0), "cfg3": (131072, 0.3, "long-range", "fast-sym", 0)}


def run(name, warm=20, steps=50):
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, PeriodicBox, SimParams, box_length_for_density
    from paper_1703_02484_b200.dynamics import LongRangeSimulation
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    from paper_1703_02484_b200.triangulation import build_initial
    n, rho, force, prec, seed = CFG[name]
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    pos, t, a, m = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=C0, seed=seed))
    sys_ = ParticleSystem(pos, t, a, m, box)
    tri = build_initial(sys_.positions, box, method="device" if n > 60000 else "host")
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01, r_cutoff=2.5 if force != "long-range" else None)
    sim = LongRangeSimulation(sys_, params, CounterRng(seed, 2), tri=tri, force=force, precision=prec)
    sim.run(warm)
    st = sim.run(steps)
    f = np.mean([s.force_ms for s in st])
    tot = np.mean([s.step_ms for s in st])
    print(f"{name}: N={n} step {tot:.4f} ms (force {f:.4f}, O(N) {tot - f:.4f}); sweeps {np.mean([s.overlap_iterations for s in st]):.1f} "
          f"flip passes {np.mean([s.flip_passes for s in st]):.1f}  [{os.environ.get('TAG', '')}]", flush=True)
    keys = [k for k in st[0].work if k.startswith("t_")]
    print("   device phase timers (us/step): " + ", ".join(
        f"{k[2:-3]} {np.mean([s.work[k] for s in st]) / 1e3:.1f}" for k in keys), flush=True)
    cnt = [k for k in st[0].work if not k.startswith("t_")]
    print("   passes/step: " + ", ".join(f"{k} {np.mean([s.work[k] for s in st]):.1f}" for k in cnt), flush=True)


for nm in sys.argv[1:]:
    run(nm)
