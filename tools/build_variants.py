"""Build kernel-variant copies of libbd_b200.so for timing experiments
(tools/time_variants.sh -> tools/time_force.py with BD_LIB_PATH=...).
Output: paper_1703_02484_b200/_lib/variants/ (not used by the product)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_02484_b200 import build  # noqa: E402

VARIANTS = {
    "sym_ct192_m2": ["BD_SY_CT=192", "BD_SY_MINB=2"],
    "sym_ct256_m1": ["BD_SY_CT=256", "BD_SY_MINB=1"],
    "sym_ct128_m3_s48": ["BD_SY_S=48"],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    out = os.path.join(os.path.dirname(build.LIB), "variants")
    with ThreadPoolExecutor(6) as ex:
        for name, path in zip(names, ex.map(lambda k: build.build(out=os.path.join(out, f"libbd_{k}.so"),
                                                                    defines=VARIANTS[k]), names)):
            print(name, path)
