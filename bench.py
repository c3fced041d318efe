"""Benchmark of the B200 Brownian-dynamics hot path (BASELINE.json metric).

Headline workload (cfg3): N = 131,072 disks, packing fraction 0.3, two-type
non-reciprocal charges c0 = [(0.5, 3, 3), (0.5, -3, -1.5)], long-range
all-pairs force + continuously maintained periodic Delaunay triangulation +
overlap correction, dt = 0.01, D = 0.01, sigma = 1 (synthetic initial state
from the reference's own init_system restatement, seed 0).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

value  = particle-steps/s = N * K / (device time of K steps), max over ranks
e2e    = the same through the public API with host buffers: every step
         uploads the positions from pinned host memory and reads back the
         positions + StepStats (host<->device copies inside the timed region)
Multi-GPU (--gpus > 1, torchrun): the all-pairs force is sharded by
receiver slice with an NCCL all-gather of positions; the O(N) path runs as
identical replicas on every rank.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1703_02484_b200.roofline import hbm_peak_gbs, phase_roofline, step_bytes  # noqa: E402

C0 = [(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)]
FLOPS_PER_PAIR = 23  # algorithmic FP64 flops per directed pair (_kernels.py:48-56)
# the symmetric evaluation's own count per directed pair: per unordered pair the
# shared geometry (min image 12, r^2 3, sqrt + mul 2, reciprocal 1) plus per
# direction alpha*w and two (mul + add) accumulations (5 x 2) = 28
SYM_FLOPS_PER_PAIR = 14
# FP64 instructions the pair kernel's inner loop executes per DIRECTED pair (SASS of the hot loop;
# DESIGN.md §3.1): fast-sym evaluates each unordered pair once (14.62 per unordered pair in the
# factored uniform loop: 256 DFMA + 130 DMUL + 82 DADD per 8 sources x 4 receivers), fast is the
# directed kernel; each instruction takes one DFMA slot of the FP64 pipe (2 flops at the measured peak)
FP64_INST_PER_PAIR = {"fast-sym": 14.875 / 2, "fast": 12.0}  # fallbacks; the ncu capture's count wins
PROFILE_ROUND = "r02"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--particles", "--n", dest="n", type=int, default=131072)
    ap.add_argument("--rho", type=float, default=0.3)
    ap.add_argument("--precision", default="auto", choices=["auto", "fast-sym", "fast", "exact"],
                    help="auto = fast-sym (Newton's third law on r^-3; sharded by block pairs + all-reduce)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-steps", type=int, default=2,
                    help="--impl reference: full steps of the real reference (baseline/_ref, numba) to time too")
    return ap.parse_args()


def workload(n, rho):
    from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    pos, types, alpha, mu = init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=C0, seed=0))
    return box, pos, types, alpha, mu


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4) if len(r) > 3 + j and r[3 + j] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def fp64_peak_tflops():
    """Measured FP64 FMA throughput of this GPU (DFMA chains, bd_probe_fp64)."""
    import ctypes
    import torch
    from paper_1703_02484_b200._lib import lib
    L = lib()
    if not hasattr(L, "bd_probe_fp64"):
        return None
    L.bd_probe_fp64.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
    L.bd_probe_fp64.restype = ctypes.c_int
    out = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")
    flops = ctypes.c_double(0)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.bd_probe_fp64(4096, ctypes.c_void_p(out.data_ptr()), st, ctypes.byref(flops))
        e1.record()
        torch.cuda.synchronize()
        best = max(best, flops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def _oracle_range_fn():
    import ctypes
    from oracle import oracle as O
    lib = O.lib()
    lib.bdo_long_range_range.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                                                   ctypes.c_int64, ctypes.c_int64,
                                                                   ctypes.c_void_p, ctypes.c_void_p]
    return lib.bdo_long_range_range


def cpu_step_sample(box, pos, alpha, mu, tri_arrays, forces, n, threads, force_pairs=1.5e9):
    """One bounded sample of the reference step on the host cores, via the C
    oracle port (kind "port"): the O(N^2) force on a slice of receivers x all
    sources (scaled to N) + one full maintenance step on all N particles
    (integrate, pass-through check, inversion repair, Lawson flips, overlap
    correction) with the given forces.  Returns (t_force_s, t_maint_s, ns)."""
    from oracle import oracle as O
    fn = _oracle_range_fn()
    ns = min(n, max(256, int(force_pairs / n)))
    out = np.empty((n, 2))
    err = np.empty(n, np.int64)
    t0 = time.perf_counter()
    fn(pos.ctypes.data, alpha.ctypes.data, mu.ctypes.data, n, float(box.length), threads, 0, ns, out.ctypes.data,
       err.ctypes.data)
    t_force = (time.perf_counter() - t0) * n / ns
    tri = O.OracleTri.from_arrays(tri_arrays, n, box.length)
    sim = O.OracleSim(pos, alpha, mu, box.length, tri=tri, force_mode=-1, seed=0, stream=2, threads=threads)
    sim.force[...] = forces
    t0 = time.perf_counter()
    st = sim.step()
    t_maint = time.perf_counter() - t0
    if st["status"] != 0:
        raise RuntimeError(f"oracle maintenance step failed: {st}")
    return t_force, t_maint, ns


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1703_02484_b200 import _abi
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, SimParams
    from paper_1703_02484_b200.dynamics import LongRangeSimulation, _decode_stats
    from paper_1703_02484_b200.triangulation import build_initial

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    gloo_test = os.environ.get("BD_BENCH_GLOO") == "1"  # multi-rank path on one GPU (validation only)
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    if world > 1:
        if gloo_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        dist.barrier()
        nccl = ".".join(map(str, torch.cuda.nccl.version())) if not gloo_test else None
        print(f"[bench] rank {rank}/{world} on cuda:{dev_index} ({torch.cuda.get_device_name(dev_index)}), "
              f"backend {dist.get_backend()}, nccl {nccl}, communicator up", file=sys.stderr, flush=True)
    n = args.n
    if args.precision == "auto":
        args.precision = "fast-sym"
    box, pos, types, alpha, mu = workload(n, args.rho)
    t_setup = time.perf_counter()
    sys_ = ParticleSystem(pos, types, alpha, mu, box)
    tri = build_initial(sys_.positions, box)
    tri0 = tri.arrays()
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01)
    kw = {}
    if world > 1:
        from paper_1703_02484_b200.distributed import ShardedLongRange
        gather = reduce = None
        if gloo_test:
            def gather(buf, mine):
                parts = [torch.empty_like(mine, device="cpu") for _ in range(world)]
                dist.all_gather(parts, mine.cpu())
                buf.copy_(torch.cat(parts, 0).to(buf.device))

            def reduce(part):
                h = part.cpu()
                dist.all_reduce(h)
                part.copy_(h.to(part.device))
        kw["sharding"] = ShardedLongRange(rank, world, gather=gather, reduce=reduce)
    sim = LongRangeSimulation(sys_, params, CounterRng(0, 2), tri=tri, precision=args.precision, **kw)
    t_setup = time.perf_counter() - t_setup
    sim.run(args.warmup)
    torch.cuda.synchronize()

    # timed region: K steps, L2 flushed (256 MiB write) before every step and
    # excluded from the device timing; events on the launching stream
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    K = args.steps
    stats_t = torch.zeros((K, _abi.STATS_WORDS), dtype=torch.int64, device="cuda")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    from paper_1703_02484_b200._lib import lib as _native
    timed_kernel = args.precision == "fast-sym"
    if timed_kernel:
        _native().bd_timing_enable(K)  # events around each launch of the pair kernel (the dominant kernel)
    if world > 1:
        dist.barrier()
    with ClockSampler(dev_index) as clk:
        torch.cuda.synchronize()
        for j in range(K):
            flush.zero_()
            ev[j][0].record()
            sim._launch_force()
            ev[j][1].record()
            sim._launch_driver(stats_t[j].data_ptr())
            ev[j][2].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    pair_ms = None
    if timed_kernel:
        import ctypes
        buf = (ctypes.c_float * K)()
        got = _native().bd_timing_read(buf, K)
        _native().bd_timing_enable(0)
        pair_ms = [float(buf[i]) for i in range(got)]
    force_ms = [ev[j][0].elapsed_time(ev[j][1]) for j in range(K)]
    maint_ms = [ev[j][1].elapsed_time(ev[j][2]) for j in range(K)]
    ms = float(sum(force_ms) + sum(maint_ms))
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        if gloo_test:
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    host_stats = [_decode_stats(r) for r in stats_t.cpu().numpy()]
    bad = [st for st in host_stats if st["status"] != 0]
    # O(N) step (persistent maintenance kernel): algorithmic bytes from its work counters vs HBM
    ne, nt = sim.tri.n_edges, sim.tri.n_triangles
    m_bytes = [step_bytes(st["work"], n, ne, nt) for st in host_stats]
    m_ms = [ev[j][1].elapsed_time(ev[j][2]) for j in range(K)]
    sim.step_index += K
    value = n * K / (ms * 1e-3)
    rep = sim.tri.audit(sim.sys.positions)

    # e2e through the public API with host buffers (positions in and out every step)
    e2e = None
    if not args.no_e2e:
        host_pos = torch.empty((n, 2), dtype=torch.float64).pin_memory()
        host_pos.copy_(sim.sys.positions_t.cpu())
        out_pos = torch.empty((n, 2), dtype=torch.float64).pin_memory()
        k2 = max(3, min(K, 10))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k2):
            sim.sys.positions_t.copy_(host_pos, non_blocking=True)
            sim.step()  # StepStats D2H inside (host sync)
            out_pos.copy_(sim.sys.positions_t, non_blocking=True)
            torch.cuda.synchronize()
            host_pos, out_pos = out_pos, host_pos  # this step's output is the next step's input
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cpu" if gloo_test else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": n * k2 / dt, "unit": "particle-steps/s", "h2d_bytes_per_step": n * 16,
               "d2h_bytes_per_step": n * 16 + 8 * _abi.STATS_WORDS, "steps": k2,
               "path": "LongRangeSimulation.step() with positions uploaded from / read back to pinned host memory"}

    failed = bool(bad) or not rep.ok
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 1 if failed else 0
    fp64 = fp64_peak_tflops()
    pairs = n * (n - 1)
    f_ms = float(np.mean(force_ms))
    achieved = FLOPS_PER_PAIR * pairs / (f_ms * 1e-3) / 1e12
    peak = fp64 if fp64 else 37.2
    cpu = None
    if world > 1:  # the CPU baseline is taken on rank 0 of the N = 1 run only
        cpu = {"value": None, "unit": "particle-steps/s", "cores": None, "kind": "port",
               "sample": "not measured at N > 1 (see the N = 1 line)"}
    elif not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            t_force, t_maint, ns = cpu_step_sample(box, pos, alpha, mu, tri0, sys_first_forces(n, pos, alpha, mu,
                                                                                               box),
                                                   n, threads)
            cpu = {"value": n / (t_force + t_maint), "unit": "particle-steps/s", "cores": threads, "kind": "port",
                   "sample": f"oracle C port of the reference step (gcc -O2 -ffp-contract=off; OpenMP {threads} "
                             f"threads for the all-pairs force like numba prange, the rest serial like the "
                             f"reference): force on {ns} of {n} receivers x all sources scaled to N "
                             f"({t_force:.2f} s) + one full maintenance step on all N ({t_maint:.3f} s)",
                   "force_s_per_step": t_force, "maintain_s_per_step": t_maint}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "particle-steps/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}
    kname = {"fast-sym": "k_allpairs_sym", "fast": "k_allpairs_fast", "exact": "k_allpairs"}[args.precision]
    traffic, pipe, inst_prof = profiled_kernel(kname, n)
    # kernels of ours per step: count + scans + scatter + in-cell sort + pack (with the tie check) + pair kernel +
    # partial sums + finish (in particle order) + rescan (fast-sym); sort (4) + pack + pair kernel + partition sums + unsort + rescan (fast); pack + pair
    # kernel (+ slot copy in / out when sharded) (exact); then the persistent step kernel
    launches_per_step = {"fast-sym": 10, "fast": 10, "exact": 3 if world == 1 else 5}[args.precision]
    inst = inst_prof or FP64_INST_PER_PAIR.get(args.precision)
    # roofline of the dominant kernel (the all-pairs pair kernel): the FP64 pipe.
    # achieved = the FP64 work the pair kernel executes per launch (FP64
    # instructions per directed pair, counted by ncu on the same kernel, x 2
    # flops per DFMA slot x N(N-1)) over its average launch time, measured
    # live with CUDA events around each launch (bd_timing_*); peak = the
    # measured DFMA throughput, so frac is the FP64-pipe fraction.  The same
    # over the whole force phase (sort, pack, tie check, partials) and the
    # algorithm's own / the reference's flop counts are reported beside it.
    k_ms = float(np.mean(pair_ms)) if pair_ms else f_ms
    hw = 2 * inst * pairs / (k_ms * 1e-3) / 1e12 if inst else None
    hw_phase = 2 * inst * pairs / (f_ms * 1e-3) / 1e12 if inst else None
    sym_flops = {"fast-sym": SYM_FLOPS_PER_PAIR}.get(args.precision, FLOPS_PER_PAIR)
    line = {
        "metric": "particle-steps/s (N x steps / s), long-range all-pairs + Delaunay maintenance + overlap correction",
        "value": None if failed else value, "unit": "particle-steps/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference init_system restatement, seed 0)",
        "config": {"workload": f"cfg3: N={n} long-range all-pairs + periodic Delaunay triangulation, rho={args.rho}, "
                               f"c0 charges, dt=0.01, D=0.01", "n": n, "rho": args.rho,
                   "precision": args.precision,
                   "parallelism": (f"allpairs-shard{world}" + ("-gloo-test" if gloo_test else "")) if world > 1
                   else "single",
                   "l2": "flushed before every timed step (256 MiB write), flush excluded from the device time"},
        "phase_ms": {"force": f_ms, "maintain": float(np.mean(maint_ms))},
        "interactions_per_s": pairs / (f_ms * 1e-3),
        "roofline": {"bound": "fp64", "achieved": hw if hw else achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (hw if hw else achieved) / peak, "traffic": traffic,
                     "peak_source": "measured DFMA probe on this GPU (bd_probe_fp64)" if fp64
                     else "nominal 148x64x2x1.965GHz",
                     "kernel": kname,
                     "kernel_ms": k_ms, "kernel_ms_source": "CUDA events around each pair-kernel launch "
                                                             "(bd_timing_enable/read)" if pair_ms else
                     "force phase events (no per-kernel timing for this precision)",
                     "fp64_inst_per_pair": inst,
                     "fp64_inst_source": "ncu sm__sass_thread_inst_executed_op_d{fma,mul,add} of the pair kernel "
                                         f"(profiles/{PROFILE_ROUND}_ncu_full_{kname}.json) / (N(N-1))"
                     if inst_prof else "SASS count of the hot loop (fallback)",
                     "fp64_pipe_active_pct_ncu": pipe,
                     "force_phase_ms": f_ms, "force_phase_achieved": hw_phase,
                     "force_phase_frac": hw_phase / peak if hw_phase else None,
                     "algorithmic_tflops": sym_flops * pairs / (k_ms * 1e-3) / 1e12,
                     "algorithmic_flops_per_directed_pair": sym_flops,
                     "reference_equiv_tflops": FLOPS_PER_PAIR * pairs / (k_ms * 1e-3) / 1e12,
                     "reference_flops_per_directed_pair": FLOPS_PER_PAIR,
                     "note": "achieved = FP64 work the pair kernel executes (fp64_inst_per_pair x 2 flops per "
                             "DFMA slot x N(N-1)) over its average launch time (kernel_ms, live CUDA events); "
                             "frac = fraction of the measured FP64 pipe peak. force_phase_* = the same over the "
                             "whole force phase. algorithmic_tflops counts the symmetric algorithm's flops (14 "
                             "per directed pair); reference_equiv_tflops the reference's 23 per directed pair "
                             "(> peak is possible: each unordered pair is evaluated once). traffic = DRAM bytes "
                             "per launch of the pair kernel (ncu --set full capture, profiles/)"},
        "maintain_roofline": {
            "bound": "hbm", "kernel": "k_step_tri_grid (persistent O(N) step)",
            "achieved": float(np.sum(m_bytes) / (np.sum(m_ms) * 1e-3) / 1e9), "unit": "GB/s",
            "peak": hbm_peak_gbs(measured_peaks()),
            "frac": float(np.sum(m_bytes) / (np.sum(m_ms) * 1e-3) / 1e9) / hbm_peak_gbs(measured_peaks()),
            "bytes_per_step": float(np.mean(m_bytes)),
            "work_per_step": {k: float(np.mean([st["work"][k] for st in host_stats])) for k in host_stats[0]["work"]},
            "phases": phase_roofline({k: float(np.mean([st["work"][k] for st in host_stats]))
                                      for k in host_stats[0]["work"]}, n, ne, nt),
            "note": "algorithmic bytes (SURVEY §8(d) per-pass minimum, paper_1703_02484_b200/roofline.py) of the "
                    "passes the kernel reports it ran, over its device time; the working set (~60 MB) is "
                    "L2-resident at this N and the kernel is grid-barrier/latency bound (profiles/)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": K * launches_per_step,
        "clocks": clk.summary(),
        "step_status_errors": len(bad),
        "audit_ok": bool(rep.ok),
        "setup_s": t_setup,
    }
    if failed:
        line["error"] = f"{len(bad)} timed steps failed (first: {bad[0] if bad else None}); audit ok: {rep.ok}"
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 1 if failed else 0


def sys_first_forces(n, pos, alpha, mu, box):
    """EXACT all-pairs forces of the initial state (bit-identical to the
    reference kernel) -- the input of the CPU maintenance-step sample."""
    from paper_1703_02484_b200 import kernels
    out, _ = kernels.long_range_kernel(pos, alpha, mu, box.length, precision="exact")
    return out


def profiled_kernel(kernel: str, n: int):
    """(DRAM bytes per launch, FP64 pipe %, FP64 instructions per directed
    pair) of `kernel` from this round's committed ncu capture (profiles/;
    made at the same N by tools/profile.sh), or Nones."""
    path = os.path.join(ROOT, "profiles", f"{PROFILE_ROUND}_ncu_full_{kernel}.json")
    try:
        for d in json.load(open(path)):
            if kernel not in d["kernel"]:
                continue

            def num(v):
                x, unit = (v.split() + [""])[:2]
                return float(x) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)

            traffic = num(d["dram_read"]) + num(d["dram_write"])
            pipe = float(d["fp64_pipe_pct"].split()[0])
            inst = None
            if "dfma_thread_inst" in d and int(d.get("n", 0)) == n:
                inst = (num(d["dfma_thread_inst"]) + num(d["dmul_thread_inst"]) + num(d["dadd_thread_inst"])) / (
                    n * (n - 1.0))
            return traffic, pipe, inst
    except Exception:
        pass
    return None, None, None


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the step on
    the host cores, as the C oracle port (kind "port": oracle/bd_oracle.c,
    the reference step restated in C with its expression order; the
    reference itself is Python and cannot be compiled into oracle/_ref).
    Every timed step is a FULL unsampled step from the evolving state: the
    all-pairs force on all N receivers (OpenMP over all host threads, like
    numba's prange in _kernels.py:37) + integrate, pass-through check,
    inversion repair, Lawson flips and overlap correction (serial, like the
    reference).  The CPU port needs no warm-up (no JIT): at most one untimed
    warm-up step is run.  When the reference package itself is installed
    under baseline/_ref, its own LongRangeSimulation (numba
    + numpy) is timed too for --ref-steps full steps, as a second stated
    baseline (`reference_numba`)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    n = args.n
    box, pos, types, alpha, mu = workload(n, args.rho)
    threads = os.cpu_count() or 1
    from paper_1703_02484_b200.core import wrap
    pos = wrap(box, pos)
    from paper_1703_02484_b200.triangulation import build_initial_arrays
    t0 = time.perf_counter()
    arrays = build_initial_arrays(pos, box)
    tri = O.OracleTri.from_arrays(arrays, n, box.length)
    tri.restore_delaunay(pos)
    t_build = time.perf_counter() - t0
    tri0 = {k: v.copy() for k, v in tri.arrays().items()}  # the port's steps mutate `tri` in place
    sim = O.OracleSim(pos, alpha, mu, box.length, tri=tri, force_mode=0, seed=0, stream=2, threads=threads)
    warm = min(args.warmup, 1)
    times = []
    for s in range(warm + args.steps):
        t0 = time.perf_counter()
        st = sim.step()
        dt = time.perf_counter() - t0
        if st["status"] != 0:
            raise RuntimeError(f"oracle step {s} failed: {st}")
        if s >= warm:
            times.append(dt)
    t_step = float(np.mean(times))
    value = n / t_step
    sample = (f"full unsampled steps of cfg3 from the evolving state: oracle C port of the reference step "
              f"(gcc -O2 -ffp-contract=off), all-pairs force on all {n} receivers with OpenMP over {threads} host "
              f"threads (numba prange in the reference), the rest serial (as the reference); {args.steps} timed "
              f"steps after {warm} untimed (no JIT to warm)")
    line = {"impl": "reference", "metric": "particle-steps/s (N x steps / s), long-range all-pairs + Delaunay "
                                           "maintenance + overlap correction",
            "value": value, "unit": "particle-steps/s", "n_gpus": args.gpus, "steps": len(times),
            "warmup": warm, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
            "config": {"workload": f"cfg3: N={n} long-range all-pairs + periodic Delaunay triangulation, "
                                   f"rho={args.rho}, c0 charges, dt=0.01, D=0.01", "n": n, "rho": args.rho},
            "dtype": "f64", "data": "synthetic (reference init_system restatement, seed 0)",
            "cpu_baseline": {"value": value, "unit": "particle-steps/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step_s": times, "setup_build_s": t_build}
    if args.ref_steps > 0:
        line["reference_numba"] = time_reference_numba(args, box, pos, types, alpha, mu, tri0, threads)
    print(json.dumps(line))


def time_reference_numba(args, box, pos, types, alpha, mu, tri0, threads):
    """The reference package itself (baseline/_ref, pip-installed from the
    reference's pkg/ with --no-deps) on its stock code path:
    brownsim.dynamics.LongRangeSimulation.step with its own numpy RngStream
    (0, 2), numba threads = all host cores.  The initial triangulation is
    the reference's (build_initial_arrays + restore_delaunay: array for
    array what brownsim.triangulation.build_initial returns, which takes
    ~25 s at this N).  Returns a stated baseline object, or why not."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "brownsim")):
        return {"unavailable": "baseline/_ref/brownsim not installed"}
    try:
        sys.path.insert(0, ref)
        import numba
        import brownsim
        from brownsim import _kernels as RK
        from brownsim.core import ParticleSystem as RPS, PeriodicBox as RBox, RngStream as RRng, SimParams as RSP
        from brownsim.dynamics import LongRangeSimulation as RLR
        from brownsim.triangulation import PeriodicTriangulation as RTri
        numba.set_num_threads(min(threads, numba.config.NUMBA_NUM_THREADS))
        # JIT warm-up: two steps of a small system compile every kernel the step uses
        t0 = time.perf_counter()
        from brownsim.initial import InitConfig as RIC, init_system as rinit
        from brownsim.core import box_length_for_density as rblen
        from brownsim.triangulation import build_initial as rbuild
        wbox = RBox(rblen(256, 1.0, 0.3))
        wsys = rinit(RIC(n=256, box=wbox, sigma=1.0, types=C0, seed=0))
        wsim = RLR(wsys, RSP(n=256, sigma=1.0, dt=0.01, diffusion=0.01), RRng(0, stream=2),
                   tri=rbuild(wsys.positions, wbox))
        wsim.step()
        wsim.step()
        t_jit = time.perf_counter() - t0
        rbox = RBox(float(box.length))
        rsys = RPS(pos.copy(), types.copy(), alpha.copy(), mu.copy(), rbox)
        rtri = RTri(rbox, pos.shape[0], **tri0)
        rsim = RLR(rsys, RSP(n=pos.shape[0], sigma=1.0, dt=0.01, diffusion=0.01), RRng(0, stream=2), tri=rtri)
        times, parts = [], []
        for _ in range(args.ref_steps):
            t0 = time.perf_counter()
            st = rsim.step()
            times.append(time.perf_counter() - t0)
            parts.append({"force_ms": st.force_ms, "maintain_ms": st.maintain_ms, "overlap_ms": st.overlap_ms})
        t = float(np.mean(times))
        return {"value": pos.shape[0] / t, "unit": "particle-steps/s", "cores": int(numba.get_num_threads()),
                "kind": "reference", "steps": len(times), "step_s": times, "phases": parts, "jit_s": t_jit,
                "sample": f"brownsim {getattr(brownsim, '__version__', '0.1.0')} LongRangeSimulation.step, "
                          f"{len(times)} full steps from the initial state after a JIT warm-up (2 steps of a 256-particle system); numba "
                          f"{numba.__version__} threads = {numba.get_num_threads()} (only the all-pairs kernel "
                          f"is threaded, the rest is numpy / Python on one core)"}
    except Exception as exc:  # pragma: no cover
        return {"unavailable": f"{type(exc).__name__}: {exc}"}


def relaunch(args):
    """--gpus N > 1 outside torchrun: start N ranks (one process per GPU)
    under torch.distributed.run on this node and return its exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    # the script's own options go after the script path; spell them out in full so that
    # torch.distributed.run's parser cannot take one for an abbreviation of its own (--n)
    own = ["--particles" if a == "--n" else ("--particles=" + a[4:] if a.startswith("--n=") else a)
           for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + own
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        sys.exit(run_ours(args))


if __name__ == "__main__":
    main()
