"""Kernel-variant builds of libbd_b200.so for FAST-SYM timing experiments
(tools/gpu_sym_iter.sh VARIANTS=...).  Output: paper_1703_02484_b200/_lib/variants/
(not used by the product).  Usage: python tools/build_sym_variants.py name=DEF1,DEF2 ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_02484_b200 import build  # noqa: E402

if __name__ == "__main__":
    specs = [a.split("=", 1) for a in sys.argv[1:]]
    out = os.path.join(os.path.dirname(build.LIB), "variants")
    jobs = [(name, [d for d in defs.split(",") if d]) for name, defs in specs]
    with ThreadPoolExecutor(len(jobs) + 1) as ex:
        futs = [ex.submit(build.build, out=os.path.join(out, f"libbd_{n}.so"), defines=d) for n, d in jobs]
        futs.append(ex.submit(build.build))
        for f in futs:
            print(f.result())
