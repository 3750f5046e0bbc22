"""BK host-array path vs the number of staging-copy threads."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import besselk as B  # noqa: E402

n = 64 << 20
rng = np.random.default_rng(20250201)
x = 140.0 * (1.0 - rng.random(n))
nu = 20.0 * (1.0 - rng.random(n))
for _ in range(3):
    bg.bessel_k_batch(x, nu)
for rep in range(2):
    for t in (2, 4, 8, 12, 16):
        B._COPY_THREADS = t
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bg.bessel_k_batch(x, nu)
            torch.cuda.synchronize()
            ts.append(round((time.perf_counter() - t0) * 1e3, 1))
        print(rep, "threads", t, sorted(ts), flush=True)
