"""Per-nu device time of the N x N Matern launch (A/B helper, GPU box).
usage: python tools/ab_nu.py [N] [nu ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import _lib  # noqa: E402
from paper_2502_00356_b200.covariance import _cov_launch, matern_plan  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
nus = [float(v) for v in sys.argv[2:]] or [0.3, 0.8, 1.7, 2.9]
locs = np.random.default_rng(20250201).random((N, 2))
lxy = torch.from_numpy(np.ascontiguousarray(locs.T)).cuda()
out = torch.empty((N, N), dtype=torch.float64, device="cuda")
res = []
for nu in nus:
    plan = matern_plan(bg.MaternParams(1.0, 0.1, nu))
    _cov_launch(plan, lxy[0], lxy[1], N, 0, N, out, N, _lib.LAYOUT_ROW_MAJOR)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        _cov_launch(plan, lxy[0], lxy[1], N, 0, N, out, N, _lib.LAYOUT_ROW_MAJOR)
    e1.record()
    torch.cuda.synchronize()
    res.append(f"nu={nu}: {e0.elapsed_time(e1) / 3:.3f} ms")
print("  ".join(res))
