"""Grid-barrier latency on this GPU: the cooperative_groups grid.sync that
ends every phase of the persistent step kernels, for their grid shapes.
Measured on a B200 (round 2): 1.23 us at 2 x 256-thread CTAs per SM, 1.63 us
at 4 per SM, 1.27 us at 1 x 1024.  A hand-written flag barrier (separate
arrival / generation words) took 2.0-2.3 us and a barrier with the phase's
sum folded into the arrival word 1.6-2.4 us: neither beats it.
Measurement only."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1703_02484_b200._lib import lib  # noqa: E402

L = lib()
scratch = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
for threads, per_sm in ((256, 1), (256, 2), (256, 4), (1024, 1)):
    best = 1e9
    for _ in range(3):
        ms = ctypes.c_double(0)
        assert L.bd_probe_barrier(iters, 0, per_sm, threads, ctypes.c_void_p(scratch.data_ptr()), st,
                                  ctypes.byref(ms)) == 0
        best = min(best, ms.value)
    print(f"{threads:5d} threads x {per_sm} CTA/SM: grid.sync {best * 1e3 / iters:.3f} us", flush=True)
