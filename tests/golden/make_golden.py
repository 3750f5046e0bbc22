"""Generate golden fixtures by importing the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box never runs this; tests only read the
committed .npz files.  The reference is imported under the alias
``besselgp_ref`` with a dedicated NUMBA_CACHE_DIR.

Every vector is produced by the reference's own kernels / public API:
  * kernels.refined_log_bessel        (kernels.py:296-302)
  * kernels.fixed_window_log_pair     (kernels.py:212-216)  bins 16/40/128
  * kernels.grid_peak_index           (kernels.py:112-123)
  * kernels.temme_sums                (kernels.py:230-270)
  * kernels.log_integrand{,_d1,_d2}   (kernels.py:52-72)
  * kernels.matern_tile               (kernels.py:338-381) with the restated
    caller's tables (h=(t1-t0)/b, c=cosh(t_m), a=log_cosh(nu t_m),
    lp=log(s2)-(nu-1)ln2-lgamma(nu))
  * besselk.bessel_k / DomainError messages (besselk.py:94-165)
"""

from __future__ import annotations

import importlib.util
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src/besselgp"
SEED = 20250201


def load_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_besselgp_ref")
    spec = importlib.util.spec_from_file_location(
        "besselgp_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["besselgp_ref"] = mod
    spec.loader.exec_module(mod)
    return mod, sys.modules["besselgp_ref.kernels"]


def bk_points(rng):
    """Seeded config vector (SURVEY 8d BK distribution) + adversarial points."""
    n = 3000
    x = 140.0 * (1.0 - rng.random(n))
    nu = 20.0 * (1.0 - rng.random(n))
    xs, nus = [x], [nu]
    # small-x (series) region
    xs.append(0.1 * (1.0 - rng.random(600)))
    nus.append(20.0 * (1.0 - rng.random(600)))
    thr = 0.1
    adv_x = [np.nextafter(thr, 0.0), thr, np.nextafter(thr, 1.0), 1e-3, 1e-8, 1e-14, 0.05, 0.09,
             0.5, 1.0, 2.0, 5.0, 10.0, 14.0, 20.0, 27.5, 30.0, 50.0, 80.0, 139.9, 140.0, 150.0,
             300.0, 700.0, 2000.0]
    adv_nu = [0.0, 1e-12, 1e-6, 0.001, 0.3, 0.5, np.nextafter(0.5, 0.0), np.nextafter(0.5, 1.0),
              1.0, 1.5, 2.0, 2.5, 2.9, 3.5, 5.0, 10.0, 16.6, 19.5, 20.0, 25.0, 40.0]
    gx, gn = np.meshgrid(np.array(adv_x), np.array(adv_nu))
    xs.append(gx.ravel())
    nus.append(gn.ravel())
    # nu^2 == x boundary (anchor switch) and half-integer +- ulp
    v = np.array([0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 7.0, 11.0])
    xs.append(v * v)
    nus.append(v)
    xs.append(np.nextafter(v * v, 0.0))
    nus.append(v)
    return np.concatenate(xs), np.concatenate(nus)


def main():
    ref, K = load_reference()
    rng = np.random.default_rng(SEED)
    eps = 2.0 ** -52
    cap = 15000

    # ---- BesselK ----------------------------------------------------------------------
    x, nu = bk_points(rng)
    refined = np.array([K.refined_log_bessel(a, b, 0.0, 9.0, 40, 0.1, eps, cap)
                        for a, b in zip(x, nu)])
    fw = {}
    mstar = {}
    for bins in (16, 40, 128):
        xi = x[x > 0]
        pairs = [K.fixed_window_log_pair(a, b, 0.0, 9.0, bins) for a, b in zip(x, nu)]
        fw[bins] = np.array([s + l for s, l in pairs])
        mstar[bins] = np.array([K.grid_peak_index(a, b, 0.0, 9.0, bins) for a, b in zip(x, nu)])
        del xi
    # a non-default window too (t_lower > 0)
    fw_shift = np.array([sum(K.fixed_window_log_pair(a, b, 0.5, 7.0, 40)) for a, b in zip(x, nu)])
    np.savez_compressed(os.path.join(HERE, "besselk.npz"), x=x, nu=nu, refined=refined,
                        fw16=fw[16], fw40=fw[40], fw128=fw[128], mstar16=mstar[16],
                        mstar40=mstar[40], mstar128=mstar[128], fw_t05_7=fw_shift)

    # ---- Temme sums -------------------------------------------------------------------
    tx = np.concatenate([0.1 * (1.0 - rng.random(400)), [1e-12, 1e-6, 0.05, np.nextafter(0.1, 0)]])
    tmu = np.concatenate([rng.random(400) - 0.5, [-0.5, 0.0, 1e-11, 0.3]])
    sums = np.array([K.temme_sums(a, b, eps, cap) for a, b in zip(tx, tmu)])
    np.savez_compressed(os.path.join(HERE, "temme.npz"), x=tx, mu=tmu, s0=sums[:, 0],
                        s1=sums[:, 1], terms=sums[:, 2].astype(np.int64))

    # ---- log integrand and derivatives --------------------------------------------------
    gt = np.concatenate([rng.random(300) * 9.0, [0.0, 1.0, 5.0, 9.0, 30.0]])
    gx = np.concatenate([rng.random(300) * 140.0 + 1e-3, [1.0, 1.0, 2.0, 4.0, 0.5]])
    gn = np.concatenate([rng.random(300) * 20.0, [0.0, 0.0, 3.0, 1.0, 50.0]])
    g0 = np.array([K.log_integrand(a, b, c) for a, b, c in zip(gt, gx, gn)])
    g1 = np.array([K.log_integrand_d1(a, b, c) for a, b, c in zip(gt, gx, gn)])
    g2 = np.array([K.log_integrand_d2(a, b, c) for a, b, c in zip(gt, gx, gn)])
    np.savez_compressed(os.path.join(HERE, "integrand.npz"), t=gt, x=gx, nu=gn, g0=g0, g1=g1,
                        g2=g2)

    # ---- Matern tiles -----------------------------------------------------------------
    N = 80
    locs = rng.random((N, 2))
    # duplicates (r == 0 off-diagonal) and very close pairs (u < thr)
    locs[7] = locs[3]
    locs[11] = locs[5] + np.array([1e-4, 0.0])
    locs[12] = locs[5] + np.array([0.0, 3e-3])
    locs[13] = locs[5] + np.array([2e-3, 2e-3])
    out = {}
    for nu_m in (0.3, 0.5, 0.8, 1.5, 1.7, 2.9):
        for beta in (0.1, 0.03):
            sigma_sq = 2.0 if nu_m == 1.7 else 1.0
            h = (9.0 - 0.0) / 40
            c = np.array([math.cosh(0.0 + m * h) for m in range(41)])
            a = np.array([K.log_cosh(nu_m * (0.0 + m * h)) for m in range(41)])
            lp = math.log(sigma_sq) - (nu_m - 1.0) * K.LN2 - math.lgamma(nu_m)
            tile = np.empty((N, N))
            K.matern_tile(tile, locs[:, 0].copy(), locs[:, 1].copy(), locs[:, 0].copy(),
                          locs[:, 1].copy(), sigma_sq, beta, nu_m, lp, c, a, h, 0.1, eps, cap)
            key = f"nu{nu_m}_beta{beta}"
            out[key] = tile
            out[key + "_lp"] = np.array([lp])
            out[key + "_s2"] = np.array([sigma_sq])
            out[key + "_c"] = c
            out[key + "_a"] = a
    np.savez_compressed(os.path.join(HERE, "matern.npz"), locs=locs, **out)

    # ---- public API (besselk.py) ------------------------------------------------------
    api_pts = [(0.05, 1.5), (2.0, 1.5), (0.1, 0.7), (1.0, 0.5), (1.0, 0.0), (0.05, 0.5),
               (140.0, 20.0), (150.0, 1.0), (1.0, 25.0), (1e-14, 20.0), (1e-300, 30.0)]
    rows = []
    for xv, nv in api_pts:
        r = ref.bessel_k(ref.EvalPoint(xv, nv))
        rows.append((xv, nv, r.log_value, r.value, 0 if r.path_taken.value == "series" else 1,
                     r.warning or ""))
    msgs = {}
    for name, fn in [("x0", lambda: ref.bessel_k(ref.EvalPoint(0.0, 1.0))),
                     ("xneg", lambda: ref.EvalPoint(-1.0, 1.0)),
                     ("nunan", lambda: ref.EvalPoint(1.0, float("nan"))),
                     ("series_big", lambda: ref.bessel_k_series(ref.EvalPoint(0.5, 1.0))),
                     ("integral_small", lambda: ref.bessel_k_integral(ref.EvalPoint(0.05, 1.0))),
                     ("temme_mu", lambda: ref.temme_pair(0.05, 0.5)),
                     ("temme_x", lambda: ref.temme_pair(0.2, 0.0)),
                     ("cfg_bins", lambda: ref.QuadratureConfig(bins=1)),
                     ("cfg_t", lambda: ref.QuadratureConfig(t_lower=9.0, t_upper=9.0)),
                     ("fw_x0", lambda: ref.fixed_window_log_bessel_k(0.0, 1.0))]:
        try:
            fn()
            msgs[name] = "<no error>"
        except Exception as e:  # noqa: BLE001
            msgs[name] = f"{type(e).__name__}: {e}"
    tp = ref.temme_pair(0.05, 0.3)
    np.savez_compressed(
        os.path.join(HERE, "api.npz"),
        x=np.array([r[0] for r in rows]), nu=np.array([r[1] for r in rows]),
        log_value=np.array([r[2] for r in rows]), value=np.array([r[3] for r in rows]),
        path=np.array([r[4] for r in rows]), warning=np.array([r[5] for r in rows]),
        err_names=np.array(list(msgs.keys())), err_msgs=np.array(list(msgs.values())),
        temme_pair_005_03=np.array(tp))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
