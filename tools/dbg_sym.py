import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from golden_io import load
from oracle import oracle as O
from paper_1703_02484_b200 import kernels
for name in ("cfg1_lr_c0_n1024", "lr_c3_n512"):
    rec = load(name)
    L = float(rec["L"])
    ref, _ = O.long_range(rec["pos0"], rec["alpha"], rec["mu"], L)
    for prec in ("fast", "fast-sym"):
        out, err = kernels.long_range_kernel(rec["pos0"], rec["alpha"], rec["mu"], L, precision=prec)
        rel = np.linalg.norm(out - ref, axis=1) / np.linalg.norm(ref, axis=1)
        i = int(rel.argmax())
        print(name, prec, "max rel", rel.max(), "at", i, "n bad", int((rel > 1e-9).sum()), "pos", rec["pos0"][i], "L/2", L / 2)
    pos = rec["pos0"]
    d = pos[:, None, :] - pos[None, :, :]
    print("exact L/2 ties x:", int((np.abs(d[..., 0]) == L / 2).sum()), "y:", int((np.abs(d[..., 1]) == L / 2).sum()))
