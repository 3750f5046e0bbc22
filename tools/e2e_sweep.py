"""M100 end to end (generate_covariance into a page-locked host array) over the host
pipeline's knobs: mirror threads and row-block size (GPU box).
usage: python tools/e2e_sweep.py [threads [block_MiB ...]]"""
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
ncpu = len(os.sched_getaffinity(0))
print("host threads", ncpu, flush=True)


def run(threads, block):
    C._MIRROR_THREADS = threads
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        bg.generate_covariance(locs, theta, out=host, host_block_bytes=block)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return ts


run(None, 1 << 30)  # warm-up
for threads in ([int(a) for a in sys.argv[1:2]] or [ncpu // 2, ncpu * 3 // 4, ncpu]):
    for block in ([int(b) << 20 for b in sys.argv[2:]] or [1 << 29, 1 << 30, 1 << 31]):
        ts = run(threads, block)
        print(f"threads {threads:3d} block {block >> 20:5d} MiB: "
              + " ".join(f"{t:.3f}" for t in ts) + f"  median {sorted(ts)[1]:.3f} s", flush=True)
