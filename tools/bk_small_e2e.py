"""Where a host-array BesselK call of 1M elements spends its time (GPU box).
usage: python tools/bk_small_e2e.py [n]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import besselk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(20250201)
x = 140.0 * (1.0 - rng.random(n))
nu = 20.0 * (1.0 - rng.random(n))


def t(fn, reps=9):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


print(f"n={n}")
print(f"bessel_k_batch(numpy)            {t(lambda: bg.bessel_k_batch(x, nu)):.2f} ms")
print(f"pipelined host path              "
      f"{t(lambda: besselk._bessel_k_host_pipelined(x, nu, bg.DEFAULT_CONFIG, 'hybrid', True)):.2f} ms")
xd = torch.from_numpy(x).cuda()
nd = torch.from_numpy(nu).cuda()
print(f"H2D pageable x + nu              {t(lambda: (torch.from_numpy(x).cuda(), torch.from_numpy(nu).cuda())):.2f} ms")
print(f"validate (device)                {t(lambda: besselk._validate_batch(xd, nd, bg.DEFAULT_CONFIG, 'hybrid')):.2f} ms")
print(f"kernel via bessel_k_batch(cuda)  {t(lambda: bg.bessel_k_batch(xd, nd, validate=False)):.2f} ms")
r = bg.bessel_k_batch(xd, nd, validate=False)
print(f"D2H pageable log K, K, path      {t(lambda: (r.log_value.cpu(), r.value.cpu(), r.path.cpu())):.2f} ms")
