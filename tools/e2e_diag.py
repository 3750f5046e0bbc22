"""Diagnose the host-buffer covariance path at N (default 100K): time the full-row
path, the lower-triangle + host-mirror path, and the host mirror alone."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import _lib, covariance as C  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
locs = np.random.default_rng(20250201).random((N, 2))
theta = bg.MaternParams(1.0, 0.1, 1.5)
host = bg.empty_host_matrix(N, N)
L = _lib.lib()


def timed(label, fn, reps=2):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label}: {min(ts):.3f} s (all {[round(t, 3) for t in ts]})", flush=True)


timed("warm", lambda: bg.generate_covariance(locs, theta, out=host), reps=1)
C._MIRROR_MIN_N = 1 << 62
timed("full rows (PCIe 80 GB)", lambda: bg.generate_covariance(locs, theta, out=host))
C._MIRROR_MIN_N = 4096
for w in [int(v) for v in os.environ.get("E2E_W", "0,4,8,12").split(",")]:
    C._MIRROR_DIRECT = w
    timed(f"lower + {w} upper blocks + host mirror", lambda: bg.generate_covariance(locs, theta, out=host))
C._MIRROR_DIRECT = None
timed("default", lambda: bg.generate_covariance(locs, theta, out=host))
nt = C._host_threads()
for t in sorted({nt, max(1, nt // 2), 2 * nt}):
    timed(f"host mirror alone, all rows, {t} threads",
          lambda: _lib.check(L.bgk_host_mirror_lower(host.ctypes.data, N, N // 2, N, t), "m"), reps=1)
