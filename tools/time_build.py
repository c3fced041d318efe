"""Initial-triangulation build times: device (build_initial(method="device"))
vs the reference construction restated on the host (method="host").
Usage: python tools/time_build.py N [rho] [seed] [--host]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1703_02484_b200.core import PeriodicBox, box_length_for_density, wrap
    from paper_1703_02484_b200.initial import InitConfig, init_arrays
    from paper_1703_02484_b200.triangulation import build_initial, build_jitter, device_build_tensors
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n = int(args[0])
    rho = float(args[1]) if len(args) > 1 else 0.3
    seed = int(args[2]) if len(args) > 2 else 0
    box = PeriodicBox(box_length_for_density(n, 1.0, rho))
    pos = wrap(box, init_arrays(InitConfig(n=n, box=box, sigma=1.0, types=[(0.5, 3.0, 3.0), (0.5, -3.0, -1.5)],
                                           seed=seed))[0])
    jit = pos + build_jitter(n, box)
    device_build_tensors(jit, box)  # warm-up (module load, allocator)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    device_build_tensors(jit, box)
    ev[1].record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    build_initial(pos, box, method="device")
    torch.cuda.synchronize()
    out = {"n": n, "rho": rho, "seed": seed, "device_build_kernel_ms": ev[0].elapsed_time(ev[1]),
           "device_build_initial_s": time.perf_counter() - t0}
    if "--host" in sys.argv:
        t0 = time.perf_counter()
        build_initial(pos, box)
        out["host_build_initial_s"] = time.perf_counter() - t0
    print(json.dumps(out))


if __name__ == "__main__":
    main()
