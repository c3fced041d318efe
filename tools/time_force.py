"""Time the all-pairs force alone (CUDA events) at N, for quick kernel iteration."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1703_02484_b200._lib import lib
from paper_1703_02484_b200 import kernels

for spec in sys.argv[1:] or ["131072:fast"]:
    n, prec = spec.split(":")
    n = int(n)
    L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
    rng = np.random.default_rng(0)
    pos = torch.from_numpy(rng.uniform(0, L, size=(n, 2))).cuda()
    t = rng.integers(0, 2, n)
    alpha = torch.from_numpy(np.where(t == 0, 3.0, -3.0)).cuda()
    mu = torch.from_numpy(np.where(t == 0, 3.0, -1.5)).cuda()
    out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    err = torch.empty(n, dtype=torch.int64, device="cuda")
    work = torch.empty(lib().bd_long_range_workspace_bytes_for(n, {"exact": 0, "fast": 1, "fast-sym": 2}[prec]) // 8 + 8, dtype=torch.int64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = {"exact": 0, "fast": 1, "fast-sym": 2}[prec]
    call = lambda: lib().bd_long_range_forces(pos.data_ptr(), alpha.data_ptr(), mu.data_ptr(), n, L, 0, n, p,
                                             out.data_ptr(), err.data_ptr(), work.data_ptr(), st)
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    reps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"n={n} {prec}: {ms:.3f} ms/force  {n*(n-1)/ms/1e9:.3f} Gpairs/ms-> {n*(n-1)/(ms*1e-3):.3e} pairs/s")

# per-rank slice of the sharded force: slots [0, n/G) of a G-way split
if os.environ.get("SLICES"):
    import ctypes as C
    from paper_1703_02484_b200 import _abi
    from paper_1703_02484_b200.core import CounterRng, ParticleSystem, PeriodicBox, SimParams
    from paper_1703_02484_b200.dynamics import make_params, _Engine
    n = 131072
    L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
    rng = np.random.default_rng(0)
    pos = rng.uniform(0, L, size=(n, 2))
    t = rng.integers(0, 2, n)
    sys_ = ParticleSystem(pos, t, np.where(t == 0, 3.0, -3.0), np.where(t == 0, 3.0, -1.5), PeriodicBox(L))
    bp = make_params(SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01), L, 0, 2, 0, 1)
    eng = _Engine(sys_, None, bp, 0)
    buf = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    lib().bd_force_prepare(C.byref(eng.s), C.byref(bp), st)
    for G in (1, 2, 4, 8):
        chunk = (n + G - 1) // G
        call = lambda: lib().bd_force_slots(C.byref(eng.s), C.byref(bp), 0, chunk, C.c_void_p(buf.data_ptr()), st)
        call(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            call()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"G={G}: per-rank slots force {ms:.3f} ms  (ideal {15.4 / G:.3f})")

# per-rank share of the sharded FAST-SYM force: bd_force_sym_partial of rank 0 of G
if os.environ.get("SYM_SLICES"):
    import ctypes as C
    from paper_1703_02484_b200 import _abi
    from paper_1703_02484_b200.core import ParticleSystem, PeriodicBox, SimParams
    from paper_1703_02484_b200.dynamics import make_params, _Engine
    n = 131072
    L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
    rng = np.random.default_rng(0)
    pos = rng.uniform(0, L, size=(n, 2))
    t = rng.integers(0, 2, n)
    sys_ = ParticleSystem(pos, t, np.where(t == 0, 3.0, -3.0), np.where(t == 0, 3.0, -1.5), PeriodicBox(L))
    bp = make_params(SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.01), L, 0, 2, 0, _abi.BD_LR_FAST_SYM)
    eng = _Engine(sys_, None, bp, 0)
    part = torch.zeros((n, 2), dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    t1 = None
    for G in (1, 2, 4, 8):
        times, ktimes = [], []
        for r in range(G):
            call = lambda: lib().bd_force_sym_partial(C.byref(eng.s), C.byref(bp), r, G, C.c_void_p(part.data_ptr()), st)
            call(); torch.cuda.synchronize()
            lib().bd_timing_enable(3)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                call()
            e1.record(); torch.cuda.synchronize()
            kb = (C.c_float * 3)()
            k = lib().bd_timing_read(kb, 3)
            lib().bd_timing_enable(0)
            times.append(e0.elapsed_time(e1) / 3)
            ktimes.append(sum(kb[i] for i in range(k)) / max(k, 1))
        t1 = t1 or times[0]
        print(f"G={G}: per-rank FAST-SYM partial (setup + pair kernel + partial sums) max {max(times):.3f} "
              f"min {min(times):.3f} ms; pair kernel alone max {max(ktimes):.3f} min {min(ktimes):.3f} ms; "
              f"force-phase efficiency T1/(G max) = {t1 / (G * max(times)):.3f}", flush=True)
