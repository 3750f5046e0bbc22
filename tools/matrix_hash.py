"""sha256 of a few Matern matrices (for bitwise A/B of library variants)."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402

h = hashlib.sha256()
for N, nu in ((3000, 1.5), (2500, 0.8), (2000, 2.9)):
    locs = np.random.default_rng(N).random((N, 2))
    m = bg.generate_covariance(locs, bg.MaternParams(1.0, 0.1, nu), device="cuda").data
    h.update(m.cpu().numpy().tobytes())
print("matrix sha256", h.hexdigest())
