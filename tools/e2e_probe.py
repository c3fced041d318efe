"""Host-side cost of the public step() on cfg3: wall time per step() vs device
time, the e2e loop with pinned host copies, the copies alone, and a cProfile
of step() (measurement only)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import bench
from paper_1703_02484_b200.core import CounterRng, ParticleSystem, SimParams
from paper_1703_02484_b200.dynamics import LongRangeSimulation
from paper_1703_02484_b200.triangulation import build_initial
n = 131072
box, pos, types, alpha, mu = bench.workload(n, 0.3)
sys_ = ParticleSystem(pos, types, alpha, mu, box)
tri = build_initial(sys_.positions, box)
sim = LongRangeSimulation(sys_, SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01), CounterRng(0, 2), tri=tri, precision="fast-sym")
sim.run(3); torch.cuda.synchronize()
K = 10
t0 = time.perf_counter()
for _ in range(K): sim.step()
t1 = time.perf_counter()
print("step() wall ms", (t1 - t0) / K * 1e3)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); sim.run(K); e1.record(); torch.cuda.synchronize(); print("run(K) device ms/step", e0.elapsed_time(e1) / K)
host_pos = torch.empty((n, 2), dtype=torch.float64).pin_memory(); host_pos.copy_(sim.sys.positions_t.cpu())
out_pos = torch.empty((n, 2), dtype=torch.float64).pin_memory()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(K):
    sim.sys.positions_t.copy_(host_pos, non_blocking=True); sim.step(); out_pos.copy_(sim.sys.positions_t, non_blocking=True); torch.cuda.synchronize(); host_pos, out_pos = out_pos, host_pos
t1 = time.perf_counter(); print("e2e loop ms/step", (t1 - t0) / K * 1e3)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(K):
    sim.sys.positions_t.copy_(host_pos, non_blocking=True); out_pos.copy_(sim.sys.positions_t, non_blocking=True); torch.cuda.synchronize()
t1 = time.perf_counter(); print("copies only ms", (t1 - t0) / K * 1e3)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5): sim.step()
pr.disable(); st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(12)
