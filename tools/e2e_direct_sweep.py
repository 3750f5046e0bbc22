"""M100 end to end over the number of upper-triangle row blocks sent directly over PCIe
next to the diagonal (covariance._MIRROR_DIRECT; 0 = host mirror only, bottom-up
blocks), with the box's host-memory copy rate for context (GPU box).
usage: python tools/e2e_direct_sweep.py [w ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import covariance as C  # noqa: E402

N = 100_000
locs = np.random.default_rng(20250201).random((N, 2))
theta = bg.MaternParams(1.0, 0.1, 1.5)
host = torch.empty((N, N), dtype=torch.float64, pin_memory=True).numpy()
a = np.ones(1 << 29)
b = np.empty_like(a)
t = time.perf_counter()
np.copyto(b, a)
print(f"host threads {len(os.sched_getaffinity(0))}, one-thread host copy "
      f"{2 * a.nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s (read + write)", flush=True)
bg.generate_covariance(locs, theta, out=host)  # warm-up
for w in [int(x) for x in sys.argv[1:]] or [0, 2, 4, 8]:
    C._MIRROR_DIRECT = w
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        bg.generate_covariance(locs, theta, out=host)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"w {w}: " + " ".join(f"{x:.3f}" for x in ts) + f"  median {sorted(ts)[1]:.3f} s",
          flush=True)
