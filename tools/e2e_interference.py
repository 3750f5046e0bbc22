"""Does the M100 host-buffer leg slow a following host-array BesselK call?  Times
bessel_k_batch on host arrays before and after an 80 GB page-locked matrix has been
filled and released."""
import gc
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402

n = 64 << 20
rng = np.random.default_rng(20250201)
x = 140.0 * (1.0 - rng.random(n))
nu = 20.0 * (1.0 - rng.random(n))


def bk(tag):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bg.bessel_k_batch(x, nu)
        torch.cuda.synchronize()
        ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    print(tag, ts, flush=True)


bk("before")
N = 100_000
locs = np.random.default_rng(1).random((N, 2))
host = bg.empty_host_matrix(N, N)
bg.generate_covariance(locs, bg.MaternParams(1.0, 0.1, 1.5), out=host)
bk("with the 80 GB matrix alive")
del host
gc.collect()
bk("after del (torch keeps the pinned block cached)")
torch._C._host_emptyCache()
bk("after host_emptyCache")
print(torch.cuda.host_memory_stats().get("allocated_bytes.current", None))
