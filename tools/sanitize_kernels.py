"""Exercise every device kernel of the library once at small sizes, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_kernels.py

Covers bgk::besselk_kernel (integral + Temme routes, ragged batch), the Matern
kernel in full row-major / column-major rows, packed lower tiles with ragged
edge tiles, explicit tiles (matern_tile), per-distance matern_batch (zero
distances, threshold entries), the audit log grid, and the location
preprocessing kernels.  Prints one line per case; exits non-zero on a failed
check (the sanitizer reports its own errors).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import audit, covariance  # noqa: E402

rng = np.random.default_rng(7)
dev = "cuda:0"

# BesselK: ragged length (not a multiple of the CTA chunk), both routes, edge values
n = 3001
x = 140.0 * (1.0 - rng.random(n))
nu = 20.0 * (1.0 - rng.random(n))
x[:50] = 0.1 * (1.0 - rng.random(50))
x[50], nu[50] = 0.1, 1e-12
x[51], nu[51] = 140.0, 20.0
r = bg.bessel_k_batch(x, nu)
assert np.all(np.isfinite(r.log_value))
print("besselk", n, "ok")

# Matern: full matrix (host and device results), a row block, lower tiles
theta = bg.MaternParams(1.0, 0.1, 1.5)
for N in (1, 37, 300):
    locs = rng.random((N, 2))
    if N > 2:
        locs[2] = locs[1]  # a duplicate location: zero distance off the diagonal
    full = bg.generate_covariance(locs, theta, device=dev).to_numpy()
    assert np.array_equal(full, full.T)
    host = bg.generate_covariance(locs, theta).to_numpy()
    assert np.array_equal(full, host)
    if N > 4:
        rows = bg.generate_covariance(locs, theta, rows=(3, N - 1), device=dev).to_numpy()
        assert np.array_equal(rows, full[3:N - 1])
    low = bg.generate_covariance(locs, bg.MaternParams(2.0, 0.07, 0.8), tile_size=64,
                                 layout="lower_tiles", device=dev)
    print("matern N=%d ok" % N)

# explicit tile / per-distance entry points
locs = rng.random((130, 2))
spec = covariance.TileSpec(0, 64, 64, 66)
t = covariance.generate_tile(spec, torch.from_numpy(locs[:64]).to(dev),
                             torch.from_numpy(locs[64:130]).to(dev), theta)
print("generate_tile ok", tuple(t.shape))
rr = np.concatenate([[0.0, 0.01, 0.1 * 0.1], 2.0 * rng.random(997)])
mv = covariance.matern_batch(rr, bg.MaternParams(1.0, 0.1, 2.9))
assert np.all(np.isfinite(np.asarray(mv.cpu() if hasattr(mv, "cpu") else mv)))
print("matern_batch ok")

# audit grid (dynamic-window oracle kernel), small
g = audit.refined_log10_grid(np.array([0.5, 3.3]), np.array([0.05, 1.0, 30.0]))
o = audit.oracle_log10_grid(np.array([0.5, 3.3]), np.array([0.05, 1.0, 30.0]), bins=1 << 10)
assert np.all(np.isfinite(g)) and np.all(np.isfinite(o))
print("audit grids ok")

# location preprocessing kernels
c = torch.from_numpy(rng.random((513, 2)) * 50.0).to(dev)
cn = covariance.normalize_locations_device(c)
covariance.morton_order_device(cn)
print("locations ok")
torch.cuda.synchronize()
print("sanitize driver done, kernel launches =", bg._lib.launch_count())
