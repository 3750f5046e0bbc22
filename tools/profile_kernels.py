"""Launch each hot kernel a few times at a profiler-friendly size (for ncu).

    python tools/profile_kernels.py matern [N] [nu]   # bgk::matern_kernel, full matrix
    python tools/profile_kernels.py besselk [n]       # bgk::besselk_kernel, BK distribution

Not a benchmark: numbers printed under a profiler are never bench values.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import _lib  # noqa: E402
from paper_2502_00356_b200.besselk import _launch_besselk  # noqa: E402
from paper_2502_00356_b200.covariance import _cov_launch, matern_plan  # noqa: E402

what = sys.argv[1]
rng = np.random.default_rng(20250201)
if what == "matern":
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    nu = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
    locs = rng.random((N, 2))
    lxy = torch.from_numpy(np.ascontiguousarray(locs.T)).cuda()
    out = torch.empty((N, N), dtype=torch.float64, device="cuda")
    plan = matern_plan(bg.MaternParams(1.0, 0.1, nu))
    for _ in range(3):
        _cov_launch(plan, lxy[0], lxy[1], N, 0, N, out, N, _lib.LAYOUT_ROW_MAJOR)
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
    x = torch.from_numpy(140.0 * (1.0 - rng.random(n))).cuda()
    nu = torch.from_numpy(20.0 * (1.0 - rng.random(n))).cuda()
    for _ in range(3):
        _launch_besselk(x, nu, bg.DEFAULT_CONFIG, _lib.ROUTE_HYBRID, want_value=True,
                        want_path=False)
torch.cuda.synchronize()
print("done", what)
