"""Phase timing probe for the cfg3 step (device events per phase, with and
without an L2 flush before the step)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1703_02484_b200 import _abi
from paper_1703_02484_b200.core import CounterRng, ParticleSystem, SimParams
from paper_1703_02484_b200.dynamics import LongRangeSimulation, _decode_stats
from paper_1703_02484_b200.triangulation import build_initial

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
prec = sys.argv[2] if len(sys.argv) > 2 else "fast-sym"
box, pos, types, alpha, mu = bench.workload(n, 0.3)
sys_ = ParticleSystem(pos, types, alpha, mu, box)
tri = build_initial(sys_.positions, box)
sim = LongRangeSimulation(sys_, SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01), CounterRng(0, 2), tri=tri,
                          precision=prec)
sim.run(3)
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
stats = torch.zeros((20, _abi.STATS_WORDS), dtype=torch.int64, device="cuda")
for do_flush in (True, False):
    fm, mm = [], []
    for j in range(10):
        if do_flush:
            flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); sim._launch_force(); e[1].record(); sim._launch_driver(stats[j].data_ptr()); e[2].record()
        torch.cuda.synchronize()
        fm.append(e[0].elapsed_time(e[1])); mm.append(e[1].elapsed_time(e[2]))
    st = [_decode_stats(r) for r in stats[:10].cpu().numpy()]
    print(f"flush={do_flush}: force {np.mean(fm):.3f} ms, maintain {np.mean(mm):.3f} ms (min {np.min(mm):.3f}); "
          f"sweeps/step {np.mean([s['overlap_iterations'] for s in st]):.1f} flip passes {np.mean([s['flip_passes'] for s in st]):.1f}")
    from paper_1703_02484_b200.roofline import phase_breakdown
    w = {k: float(np.mean([s['work'][k] for s in st])) for k in st[0]['work']}
    print("   work/step:", {k: round(v, 1) for k, v in w.items()})
    print("   time shares:", {k: round(v, 3) for k, v in phase_breakdown(w).items()})
    from paper_1703_02484_b200.roofline import phase_roofline
    print("   phase GB/s:", {k: round(v["GBs"]) for k, v in phase_roofline(w, n, sim.tri.n_edges, sim.tri.n_triangles).items()})
# host-side launch cost of the driver
t0 = time.perf_counter()
for j in range(10):
    sim._launch_driver(stats[j].data_ptr())
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue of the driver launch: {(t1 - t0) / 10 * 1e3:.3f} ms")
