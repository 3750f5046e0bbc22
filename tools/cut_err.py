"""Max relative error of the Matern matrix against the CPU oracle for the installed
library (A/B of plan options that change values, e.g. the window cutoff).
usage: python tools/cut_err.py [N]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import oracle as orc  # noqa: E402
import paper_2502_00356_b200 as bg  # noqa: E402

orc.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
worst = 0.0
for nu in (0.3, 0.8, 1.5, 1.7, 2.9, 5.3, 19.5):
    locs = np.random.default_rng(int(nu * 10)).random((N, 2))
    cov = bg.generate_covariance(locs, bg.MaternParams(1.0, 0.1, nu), device="cuda").to_numpy()
    ref = orc.generate_covariance(locs, 1.0, 0.1, nu, threads=16)
    e = float(np.max(np.abs(cov - ref) / np.maximum(np.abs(ref), 1e-300)))
    worst = max(worst, e)
    print(f"nu={nu} max rel err {e:.3e}")
print(f"worst {worst:.3e}")
