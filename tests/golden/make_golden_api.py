"""Golden vectors for the scalar drop-in API, made by the REFERENCE's own public
functions (besselk.py:94-165): bessel_k_series, bessel_k_integral,
fixed_window_log_bessel_k (default bins and the ``bins=`` override, default and
non-default QuadratureConfig) and temme_pair.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_api.py

Writes tests/golden/api_paths.npz; the GPU tests only read it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import load_reference  # noqa: E402


def main():
    ref, _ = load_reference()
    cfgs = {"default": ref.QuadratureConfig(),
            "wide": ref.QuadratureConfig(t_lower=0.0, t_upper=12.0, bins=96,
                                         small_x_threshold=0.05)}
    out = {}
    # bessel_k_series: 0 < x < threshold (besselk.py:104-110)
    ser = [(0.05, 1.5), (1e-3, 0.3), (0.0999, 7.25), (1e-8, 19.9), (0.02, 0.0), (0.07, 12.5)]
    # bessel_k_integral: x >= threshold (besselk.py:149-155)
    itg = [(0.1, 0.7), (1.0, 0.5), (2.0, 1.5), (14.1, 2.9), (50.0, 10.0), (140.0, 20.0),
           (150.0, 1.0), (1.0, 25.0), (700.0, 3.0)]
    for cname, cfg in cfgs.items():
        thr = cfg.small_x_threshold
        rows = []
        for xv, nv in ser:
            if xv < thr:
                r = ref.bessel_k_series(ref.EvalPoint(xv, nv), cfg)
                rows.append((xv, nv, r.log_value, r.value, r.warning or ""))
        out[f"series_{cname}"] = rows
        rows = []
        for xv, nv in itg:
            if xv >= thr:
                r = ref.bessel_k_integral(ref.EvalPoint(xv, nv), cfg)
                rows.append((xv, nv, r.log_value, r.value, r.warning or ""))
        out[f"integral_{cname}"] = rows
    # fixed_window_log_bessel_k: no threshold guard, bins override (besselk.py:134-146)
    fw_pts = [(1e-3, 1.5), (0.05, 0.5), (0.5, 2.0), (3.0, 0.3), (14.0, 5.0), (80.0, 16.6),
              (140.0, 0.5)]
    fw = []
    for cname, cfg in cfgs.items():
        for bins in (None, 16, 128):
            for xv, nv in fw_pts:
                v = ref.fixed_window_log_bessel_k(xv, nv, cfg, bins=bins)
                fw.append((cname, -1 if bins is None else bins, xv, nv, v))
    tp = []
    for cname, cfg in cfgs.items():
        for xv, mu in [(0.05, 0.3), (0.01, -0.5), (0.04, 0.0), (1e-6, 0.4999), (0.049, -0.2)]:
            if xv < cfg.small_x_threshold:
                k0, k1 = ref.temme_pair(xv, mu, cfg)
                tp.append((cname, xv, mu, k0, k1))

    arrays = {}
    for key, rows in out.items():
        arrays[key + "_x"] = np.array([r[0] for r in rows])
        arrays[key + "_nu"] = np.array([r[1] for r in rows])
        arrays[key + "_log_value"] = np.array([r[2] for r in rows])
        arrays[key + "_value"] = np.array([r[3] for r in rows])
        arrays[key + "_warning"] = np.array([r[4] for r in rows])
    arrays["fw_cfg"] = np.array([r[0] for r in fw])
    arrays["fw_bins"] = np.array([r[1] for r in fw], dtype=np.int64)
    arrays["fw_x"] = np.array([r[2] for r in fw])
    arrays["fw_nu"] = np.array([r[3] for r in fw])
    arrays["fw_log_value"] = np.array([r[4] for r in fw])
    arrays["tp_cfg"] = np.array([r[0] for r in tp])
    arrays["tp_x"] = np.array([r[1] for r in tp])
    arrays["tp_mu"] = np.array([r[2] for r in tp])
    arrays["tp_k0"] = np.array([r[3] for r in tp])
    arrays["tp_k1"] = np.array([r[4] for r in tp])
    np.savez_compressed(os.path.join(HERE, "api_paths.npz"), **arrays)
    print("wrote", os.path.join(HERE, "api_paths.npz"))


if __name__ == "__main__":
    main()
