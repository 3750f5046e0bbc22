"""Max |d ln K| of the GPU BesselK batch vs the CPU oracle over the BK config's first
n points (default 1M) plus adversarial grids.  usage: python tools/bk_maxerr.py [n]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402  (checker)

import paper_2502_00356_b200 as bg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
rng = np.random.default_rng(20250201)
x = 140.0 * (1.0 - rng.random(n))
nu = 20.0 * (1.0 - rng.random(n))
gx, gn = np.meshgrid(np.geomspace(0.1, 140.0, 700), np.linspace(0.0, 20.0, 400))
x = np.concatenate([x, gx.ravel()])
nu = np.concatenate([nu, gn.ravel()])
got = bg.bessel_k_batch(x, nu).log_value
ref = oracle.refined_log_bessel_batch(x, nu)
d = np.abs(got - ref)
i = int(np.argmax(d))
print(f"n={x.size} max|dlnK|={d.max():.3e} at x={x[i]!r} nu={nu[i]!r}; "
      f"p99.99={np.quantile(d, 0.9999):.2e} mean={d.mean():.2e}")
