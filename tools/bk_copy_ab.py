"""A/B the staging copy of the host-array BesselK path: native NT copy vs numpy threads."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import besselk as B  # noqa: E402

n = 64 << 20
rng = np.random.default_rng(20250201)
x = 140.0 * (1.0 - rng.random(n))
nu = 20.0 * (1.0 - rng.random(n))
native = B._par_copy
pool = ThreadPoolExecutor(16)


def numpy_copy(dst, src):
    step = max(1 << 16, -(-src.size // 16))
    for f in [pool.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, src.size, step)]:
        f.result()


for rep in range(3):
    for name, fn in (("native", native), ("numpy16", numpy_copy)):
        B._par_copy = fn
        ts = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bg.bessel_k_batch(x, nu, validate=False)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(rep, name, [round(t * 1e3, 1) for t in ts[1:]], flush=True)
