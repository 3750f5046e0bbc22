"""Golden fixtures for the GPU accuracy audit, from the REFERENCE's own oracle.py.

    python tests/golden/make_golden_audit.py     (build container only)

Writes tests/golden/audit.npz:
  * oracle_log_bessel_k (2^16 bins) at seeded + edge points      (oracle.py:137-151)
  * oracle_log10_grid (2^14 bins), refined_log10_grid, pure_integral_log10_grid
    on small (nu, x) grids incl. x < 0.1                           (oracle.py:194-217,
                                                                   kernels.py:306-329)
  * the Algorithm-1 AE curve over SPEC's region grid, bins 2^12
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402


def main():
    ref, K = load_reference()
    O = sys.modules["besselgp_ref.oracle"] if "besselgp_ref.oracle" in sys.modules else None
    if O is None:
        import importlib

        O = importlib.import_module("besselgp_ref.oracle")
    rng = np.random.default_rng(4242)
    # --- oracle points ---
    x = np.concatenate([140.0 * (1.0 - rng.random(40)), 0.1 + 2.0 * rng.random(10),
                        [0.1, 1.0, 10.0, 50.0, 139.0, 0.05, 0.01]])
    nu = np.concatenate([20.0 * (1.0 - rng.random(50)), [0.5, 3.0, 20.0, 0.001, 7.0, 2.0, 0.3]])
    olog = np.array([O.oracle_log_bessel_k(ref.EvalPoint(a, b)) for a, b in zip(x, nu)])
    # --- grids ---
    gn = np.array([0.001, 0.3, 0.5, 1.0, 2.5, 7.0, 12.0, 20.0])
    gx = np.array([0.001, 0.05, 0.1, 0.7, 3.0, 14.0, 60.0, 140.0])
    o10 = O.oracle_log10_grid(gn, gx, bins=2 ** 14)
    hn = np.linspace(0.01, 20.0, 12)
    hx = np.concatenate([[0.002, 0.04, 0.099], np.linspace(0.1, 140.0, 9)])
    r10 = np.empty((hn.size, hx.size))
    p10 = np.empty((hn.size, hx.size))
    cfg = ref.QuadratureConfig()
    K.refined_log10_grid(hn, hx, 0.0, 9.0, 40, 0.1, cfg.eps_machine, cfg.series_cap, r10)
    K.pure_integral_log10_grid(hn, hx, 0.0, 9.0, 40, p10)
    # --- Algorithm 1 curve (reference primitives) ---
    xs = np.linspace(0.0, 140.0, 141)
    xs[0] = 0.1
    xs = np.unique(np.concatenate([xs, np.geomspace(0.1, 1.0, 50)]))
    nus = np.linspace(0.5, 20.0, 40)
    oref = np.array([[O.oracle_log_bessel_k(ref.EvalPoint(a, b), bins=2 ** 12) for a in xs]
                     for b in nus])
    curve = []
    for L in (5, 6, 7, 8, 9, 10, 11, 12):
        fw = np.array([[sum(K.fixed_window_log_pair(a, b, 0.0, float(L), 2 ** 12)) for a in xs]
                       for b in nus])
        curve.append(float(np.max(np.abs(oref - fw))))
    np.savez_compressed(os.path.join(HERE, "audit.npz"), x=x, nu=nu, oracle_log=olog, gn=gn,
                        gx=gx, oracle_log10_2p14=o10, hn=hn, hx=hx, refined_log10=r10,
                        pure_integral_log10=p10, bound_L=np.arange(5, 13, dtype=float),
                        bound_ae=np.array(curve), bound_oracle_2p12=oref, bound_xs=xs,
                        bound_nus=nus)
    print("audit fixtures written; bound curve", curve)


if __name__ == "__main__":
    main()
