"""GPU parity of the BesselK kernels (bgk_besselk_batch & friends) against the
reference (golden fixtures) and the CPU oracle.

Tolerance (BASELINE.json north_star): max relative error of K <= 1e-10, i.e.
|ln K_gpu - ln K_ref| <= 1e-10 (relative error of K == absolute error of ln K).
Measured margins are far tighter (~1e-13); the asserts use 1e-10.
"""

import math

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def bg():
    import paper_2502_00356_b200 as bg

    return bg


def _lnk(bg, x, nu, route="hybrid", cfg=None):
    cfg = cfg or bg.DEFAULT_CONFIG
    return bg.bessel_k_batch(np.asarray(x), np.asarray(nu), cfg, route=route, validate=False)


def test_golden_refined(bg, golden):
    g = golden("besselk")
    r = _lnk(bg, g["x"], g["nu"])
    ref = g["refined"]
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(r.log_value), fin)
    assert np.max(np.abs(r.log_value[fin] - ref[fin])) <= TOL
    # path codes follow the strict x < threshold rule (kernels.py:299)
    assert np.array_equal(r.path, np.where(g["x"] < 0.1, 0, 1).astype(np.uint8))
    # value == exp(log_value) with overflow -> inf
    with np.errstate(over="ignore"):
        assert np.array_equal(r.value, np.exp(r.log_value)) or np.max(
            rel_err(r.value, np.exp(r.log_value))) <= 4e-16


# The unguarded integral route (fixed_window_log_bessel_k) is compared with the
# reference over the paper's audit range x >= 1e-3.  Below it the
# reference's rebase onto t_hat = asinh(nu/x) >> t_upper (kernels.py:197-209)
# cancels catastrophically (terms ~1e18 for a result ~10): its value carries
# libm-rounding noise up to ~4e-6, so no other libm can reproduce it.  There the
# kernel is checked against the exact fixed-grid sum instead (mpmath).
AUDIT_X_MIN = 1e-3


@pytest.mark.parametrize("bins", [16, 40, 128])
def test_golden_fixed_window_bins(bg, golden, bins):
    g = golden("besselk")
    cfg = bg.QuadratureConfig(bins=bins)
    r = _lnk(bg, g["x"], g["nu"], route="integral", cfg=cfg)
    ref = g[f"fw{bins}"]
    sel = np.isfinite(ref) & (g["x"] >= AUDIT_X_MIN)
    assert np.max(np.abs(r.log_value[sel] - ref[sel])) <= TOL


def test_golden_shifted_window(bg, golden):
    g = golden("besselk")
    cfg = bg.QuadratureConfig(t_lower=0.5, t_upper=7.0)
    r = _lnk(bg, g["x"], g["nu"], route="integral", cfg=cfg)
    ref = g["fw_t05_7"]
    sel = np.isfinite(ref) & (g["x"] >= AUDIT_X_MIN)
    assert np.max(np.abs(r.log_value[sel] - ref[sel])) <= TOL


@pytest.mark.parametrize("bins", [16, 40])
def test_integral_route_tiny_x_vs_exact_sum(bg, bins):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 40
    xs = [1e-14, 1e-8, 1e-5]
    nus = [0.3, 1.5, 3.5, 10.0]
    X, NU = np.meshgrid(xs, nus)
    cfg = bg.QuadratureConfig(bins=bins)
    r = _lnk(bg, X.ravel(), NU.ravel(), route="integral", cfg=cfg)
    H = mpmath.mpf(9) / bins
    for v, x, nu in zip(r.log_value, X.ravel(), NU.ravel()):
        s = sum((mpmath.mpf(0.5) if k in (0, bins) else 1) * mpmath.cosh(nu * k * H)
                * mpmath.exp(-x * mpmath.cosh(k * H)) for k in range(bins + 1))
        assert abs(v - float(mpmath.log(H * s))) <= 1e-12 * max(1.0, abs(v))


def test_series_route_matches_oracle(bg, oracle):
    rng = np.random.default_rng(7)
    x = 0.1 * (1.0 - rng.random(4000))
    nu = 25.0 * rng.random(4000)
    r = _lnk(bg, x, nu, route="series")
    ref = np.array([oracle.temme_series_log(a, b) for a, b in zip(x, nu)])
    assert np.max(np.abs(r.log_value - ref)) <= TOL


def test_bk_config_distribution_vs_oracle(bg, oracle):
    """The BK bench distribution, 1M points vs the threaded oracle."""
    rng = np.random.default_rng(20250201)
    n = 1_000_000
    x = 140.0 * (1.0 - rng.random(n))
    nu = 20.0 * (1.0 - rng.random(n))
    r = _lnk(bg, x, nu)
    ref = oracle.refined_log_bessel_batch(x, nu, threads=8)
    err = np.abs(r.log_value - ref)
    assert np.max(err) <= TOL, (np.max(err), x[np.argmax(err)], nu[np.argmax(err)])


def test_edge_inputs(bg, oracle):
    thr = 0.1
    xs = [np.nextafter(thr, 0), thr, np.nextafter(thr, 1), 1e-300, 1e-14, 1e-3, 0.5, 1.0,
          139.999, 140.0, 150.0, 700.0, 5000.0, 1e5]
    nus = [0.0, 1e-300, 1e-12, 0.5, np.nextafter(0.5, 0), 1.0, 2.0, 19.999, 20.0, 35.0, 70.0, 100.0]
    X, NU = np.meshgrid(xs, nus)
    X, NU = X.ravel(), NU.ravel()
    r = _lnk(bg, X, NU)
    ref = oracle.refined_log_bessel_batch(X, NU)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(r.log_value), fin)
    err = np.abs(r.log_value[fin] - ref[fin])
    assert np.max(err) <= TOL * np.maximum(1.0, np.abs(ref[fin])).max()
    # relative form where |ln K| is huge (x -> 0 with large nu)
    assert np.max(err / np.maximum(1.0, np.abs(ref[fin]))) <= TOL


def test_empty_and_broadcast(bg):
    r = bg.bessel_k_batch(np.zeros(0), np.zeros(0))
    assert r.log_value.shape == (0,)
    r2 = bg.bessel_k_batch(np.array([[1.0, 2.0], [3.0, 4.0]]), 1.5)
    assert r2.log_value.shape == (2, 2)
    for (i, j), xv in np.ndenumerate(np.array([[1.0, 2.0], [3.0, 4.0]])):
        k = math.sqrt(math.pi / (2 * xv)) * math.exp(-xv) * (1 + 1 / xv)
        assert abs(r2.value[i, j] / k - 1) < 1e-7


def test_batch_independent_of_size_and_order(bg):
    rng = np.random.default_rng(3)
    x = 140.0 * (1.0 - rng.random(50_000))
    nu = 20.0 * (1.0 - rng.random(50_000))
    x[::97] = 0.05 * rng.random(x[::97].size) + 1e-6
    full = _lnk(bg, x, nu).log_value
    perm = rng.permutation(x.size)
    again = _lnk(bg, x[perm], nu[perm]).log_value
    assert np.array_equal(full[perm], again)  # bitwise: pure function of (x, nu)
    part = _lnk(bg, x[:777], nu[:777]).log_value
    assert np.array_equal(part, full[:777])


def test_device_tensors_roundtrip(bg):
    import torch

    # x <= 14: where the reference discretisation itself is < 1e-10 off
    x = torch.linspace(0.05, 14.0, 1000, dtype=torch.float64, device="cuda")
    nu = torch.full_like(x, 2.5)
    r = bg.bessel_k_batch(x, nu)
    assert r.log_value.is_cuda and r.path.dtype == torch.uint8
    xv = x.cpu().numpy()
    closed = np.log(np.sqrt(np.pi / (2 * xv)) * np.exp(-xv) * (1 + 3 / xv + 3 / xv ** 2))
    assert np.max(np.abs(r.log_value.cpu().numpy() - closed)) < 1e-9


def test_temme_sums_batch(bg, golden):
    g = golden("temme")
    s0, s1, terms = bg.temme_sums_batch(g["x"], g["mu"])
    assert np.array_equal(terms, g["terms"])
    assert np.max(rel_err(s0, g["s0"])) <= 1e-13
    assert np.max(rel_err(s1, g["s1"])) <= 1e-13


def test_log_integrand_family(bg, golden):
    g = golden("integrand")
    for i in range(0, g["t"].size, 5):
        p = bg.EvalPoint(float(g["x"][i]), float(g["nu"][i]))
        t = float(g["t"][i])
        for fn, key in ((bg.log_integrand, "g0"), (bg.log_integrand_d1, "g1"),
                        (bg.log_integrand_d2, "g2")):
            v = fn(t, p)
            ref = float(g[key][i])
            assert abs(v - ref) <= 1e-13 * max(1.0, abs(ref)), (key, i, v, ref)


def test_host_pipeline_matches_device_path(bg):
    """Large numpy batches take the chunked pinned pipeline; same bits as device tensors."""
    import torch

    from paper_2502_00356_b200 import besselk as bk

    rng = np.random.default_rng(21)
    n = bk._HOST_CHUNK * 2 + 12345
    x = 140.0 * (1.0 - rng.random(n))
    nu = 20.0 * (1.0 - rng.random(n))
    x[::1001] = 0.05 * (1.0 - rng.random(x[::1001].size))
    host = bg.bessel_k_batch(x, nu, validate=True)
    dev = bg.bessel_k_batch(torch.from_numpy(x).cuda(), torch.from_numpy(nu).cuda())
    assert isinstance(host.log_value, np.ndarray)
    assert np.array_equal(host.log_value, dev.log_value.cpu().numpy())
    assert np.array_equal(host.value, dev.value.cpu().numpy())
    assert np.array_equal(host.path, dev.path.cpu().numpy())
    with pytest.raises(bg.DomainError):
        bad = x.copy()
        bad[n - 5] = -1.0
        bg.bessel_k_batch(bad, nu)
    # deferred validation reports the FIRST offending element with its own message
    bad = x.copy()
    bad[n // 2] = -1.0
    badnu = nu.copy()
    badnu[n // 3] = np.nan
    with pytest.raises(bg.DomainError) as first:
        bg.bessel_k_batch(bad, badnu)
    with pytest.raises(bg.DomainError) as single:
        bg.EvalPoint(float(x[n // 3]), float("nan"))
    assert str(first.value) == str(single.value)


def test_wide_domain_vs_oracle(bg, oracle):
    """Beyond the BK configuration: x log-uniform over [0.1, 1e4] and nu over [0, 60]
    (the fast path's window table covers x up to 2^10; larger x take the full grid).
    The folded node exponent's running bracket x c_a + nu (t_k - t_a) rounds at
    ulp(x c_a) per node, so its error grows with x; it stays far inside the tolerance."""
    rng = np.random.default_rng(7)
    n = 200_000
    x = 10.0 ** rng.uniform(-1.0, 4.0, n)
    nu = 60.0 * rng.random(n)
    r = _lnk(bg, x, nu)
    ref = oracle.refined_log_bessel_batch(x, nu, threads=8)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(r.log_value), fin)
    err = np.abs(r.log_value[fin] - ref[fin]) / np.maximum(1.0, np.abs(ref[fin]))
    assert np.max(err) <= TOL, (np.max(err), x[fin][np.argmax(err)], nu[fin][np.argmax(err)])
