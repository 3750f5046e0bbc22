"""Pin the CPU oracle (oracle/besselgp_oracle.c) against golden vectors produced by
importing the reference package itself (tests/golden/make_golden.py).

The oracle is a line-by-line C restatement of kernels.py compiled without fp
contraction, so it is expected to be BITWISE equal to the numba reference on
the integral path; the Temme path is allowed a few ulp (glibc tgamma vs the
numba gamma) but in practice is bitwise too.
"""

import math

import numpy as np
import pytest

from conftest import rel_err


def test_refined_log_bessel_bitwise(oracle, golden):
    g = golden("besselk")
    out = oracle.refined_log_bessel_batch(g["x"], g["nu"], threads=4)
    finite = np.isfinite(g["refined"])
    assert np.array_equal(np.isfinite(out), finite)
    # bitwise on every finite point
    assert np.array_equal(out[finite], g["refined"][finite])


@pytest.mark.parametrize("bins", [16, 40, 128])
def test_fixed_window_pair_and_peak_bitwise(oracle, golden, bins):
    g = golden("besselk")
    x, nu = g["x"], g["nu"]
    sel = np.arange(0, x.size, 7)  # every 7th point keeps the pure-python loop fast
    fw = np.array([sum(oracle.fixed_window_log_pair(x[i], nu[i], 0.0, 9.0, bins)) for i in sel])
    ref = g[f"fw{bins}"][sel]
    ok = np.isfinite(ref)
    assert np.array_equal(fw[ok], ref[ok])
    ms = np.array([oracle.grid_peak_index(x[i], nu[i], 0.0, 9.0, bins) for i in sel])
    assert np.array_equal(ms, g[f"mstar{bins}"][sel])


def test_fixed_window_shifted_window(oracle, golden):
    g = golden("besselk")
    x, nu = g["x"], g["nu"]
    sel = np.arange(0, x.size, 11)
    fw = np.array([sum(oracle.fixed_window_log_pair(x[i], nu[i], 0.5, 7.0, 40)) for i in sel])
    ref = g["fw_t05_7"][sel]
    ok = np.isfinite(ref)
    assert np.array_equal(fw[ok], ref[ok])


def test_temme_sums(oracle, golden):
    g = golden("temme")
    for i in range(g["x"].size):
        s0, s1, terms = oracle.temme_sums(g["x"][i], g["mu"][i])
        assert terms == g["terms"][i]
        assert rel_err(s0, g["s0"][i]) <= 4e-16
        assert rel_err(s1, g["s1"][i]) <= 4e-16


def test_log_integrand_family(oracle, golden):
    g = golden("integrand")
    for i in range(g["t"].size):
        t, x, nu = g["t"][i], g["x"][i], g["nu"][i]
        assert oracle.log_integrand(t, x, nu) == g["g0"][i]
        assert oracle.log_integrand_d1(t, x, nu) == g["g1"][i]
        assert oracle.log_integrand_d2(t, x, nu) == g["g2"][i]


def test_matern_tile_bitwise(oracle, golden):
    g = golden("matern")
    locs = g["locs"]
    keys = [k for k in g.files if k.startswith("nu") and "_" in k and k.count("_") == 1]
    assert len(keys) == 12
    for key in keys:
        nu = float(key.split("_")[0][2:])
        beta = float(key.split("_")[1][4:])
        c, a, h = oracle.matern_tables(nu)
        assert np.array_equal(c, g[key + "_c"]) and np.array_equal(a, g[key + "_a"])
        tile = oracle.matern_tile(locs[:, 0], locs[:, 1], locs[:, 0], locs[:, 1],
                                  float(g[key + "_s2"][0]), beta, nu, float(g[key + "_lp"][0]),
                                  c, a, h)
        assert np.array_equal(tile, g[key]), key


def test_generate_covariance_restated_caller(oracle, golden):
    """The restated caller (lower tiles + mirror) equals entrywise matern_tile for
    several tile sizes (SPEC.md:335 tile/scalar equivalence)."""
    g = golden("matern")
    locs = g["locs"]
    key = "nu1.5_beta0.1"
    lp = oracle.matern_log_prefactor(1.0, 1.5)
    assert abs(lp - float(g[key + "_lp"][0])) <= 1e-15  # glibc vs CPython lgamma: <= 1 ulp
    ref = g[key]
    for ts in (1, 7, 64, 256):
        full = oracle.generate_covariance(locs, 1.0, 0.1, 1.5, tile_size=ts, threads=2)
        # lp from glibc lgamma may differ from CPython's by an ulp
        assert np.max(rel_err(full, ref)) <= 1e-15, ts
        assert np.array_equal(full, full.T)
    rows = oracle.generate_covariance(locs, 1.0, 0.1, 1.5, tile_size=7, row_range=(13, 41))
    full = oracle.generate_covariance(locs, 1.0, 0.1, 1.5, tile_size=7)
    assert np.array_equal(rows, full[13:41])


def test_oracle_closed_forms(oracle):
    """Sanity of the oracle against exact half-integer closed forms where the
    reference discretisation is accurate (x <= 14)."""
    for nu in (0.5, 1.5, 2.5):
        for x in np.geomspace(0.1, 14.0, 25):
            lk = oracle.refined_log_bessel(x, nu)
            assert abs(lk - math.log(oracle.k_half_integer(x, nu))) < 1e-9
        for x in np.geomspace(1e-4, 0.099, 10):
            lk = oracle.refined_log_bessel(x, nu)
            assert abs(lk - math.log(oracle.k_half_integer(x, nu))) < 1e-10
