"""M100 host-buffer path vs the number of mirror threads."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import covariance as C  # noqa: E402

N = 100_000
locs = np.random.default_rng(1).random((N, 2))
host = bg.empty_host_matrix(N, N)
th = bg.MaternParams(1.0, 0.1, 1.5)
bg.generate_covariance(locs, th, out=host)
for rep in range(2):
    for t in (4, 6, 8, 12, 16):
        C._MIRROR_THREADS = t
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bg.generate_covariance(locs, th, out=host)
            torch.cuda.synchronize()
            ts.append(round(time.perf_counter() - t0, 3))
        print(rep, "threads", t, ts, flush=True)
