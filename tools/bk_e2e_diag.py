"""Diagnose the host-array BesselK path (64Mi elements): whole call vs its parts."""
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


def timed(label, fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label}: {min(ts) * 1e3:.1f} ms (all {[round(t * 1e3, 1) for t in ts]})", flush=True)


timed("bessel_k_batch host arrays", lambda: bg.bessel_k_batch(x, nu, validate=False))
for th in (8, 16):
    B._COPY_THREADS = th
    timed(f"  same, {th} copy threads", lambda: bg.bessel_k_batch(x, nu, validate=False))
pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
for th in (8, 16):
    B._COPY_THREADS = th
    timed(f"staging copy x only (512 MB), {th} threads", lambda: B._par_copy(pin, x))
dx = torch.empty(n, dtype=torch.float64, device="cuda")
pt = torch.from_numpy(pin)
timed("H2D 512 MB pinned", lambda: dx.copy_(pt, non_blocking=True))
timed("D2H 512 MB pinned", lambda: pt.copy_(dx, non_blocking=True))
timed("alloc 3 pinned outputs", lambda: [torch.empty(n, dtype=torch.float64, pin_memory=True),
                                         torch.empty(n, dtype=torch.float64, pin_memory=True),
                                         torch.empty(n, dtype=torch.uint8, pin_memory=True)])
# full duplex?  H2D and D2H of 512 MB each on two streams at once
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dy = torch.empty(n, dtype=torch.float64, device="cuda")
pin2 = torch.empty(n, dtype=torch.float64, pin_memory=True)


def duplex():
    with torch.cuda.stream(s1):
        dx.copy_(pt, non_blocking=True)
    with torch.cuda.stream(s2):
        pin2.copy_(dy, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


timed("H2D + D2H 512 MB each, two streams", duplex)
# the pipelined call's own timeline, chunk by chunk (events on its streams)
import paper_2502_00356_b200.besselk as BB  # noqa: E402
t0 = time.perf_counter()
r = bg.bessel_k_batch(x, nu, validate=False)
print(f"call {1e3 * (time.perf_counter() - t0):.1f} ms")
