"""Run the all-pairs force kernel alone (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1703_02484_b200 import kernels

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
prec = sys.argv[2] if len(sys.argv) > 2 else "fast"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
L = float(np.sqrt(n * np.pi * 0.25 / 0.3))
rng = np.random.default_rng(0)
pos = rng.uniform(0, L, size=(n, 2))
t = rng.integers(0, 2, n)
alpha = np.where(t == 0, 3.0, -3.0)
mu = np.where(t == 0, 3.0, -1.5)
for _ in range(reps):
    out, err = kernels.long_range_kernel(pos, alpha, mu, L, precision=prec)
torch.cuda.synchronize()
print("ok", out[:2], err.max())
