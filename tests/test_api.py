"""CPU tests of the Python boundary: same names, validation and messages as the
reference (besselk.py, __init__.py; messages pinned by tests/golden/api.npz made
from the reference itself), the SPEC covariance types and host-side helpers,
and the no-CPU-fallback rule (numeric calls fail loudly without a GPU)."""

import math
import os

import numpy as np
import pytest
import torch

import paper_2502_00356_b200 as bg


def test_public_names_cover_reference():
    ref_names = ["BesselResult", "DomainError", "EvalPoint", "PathTaken", "QuadratureConfig",
                 "bessel_k", "bessel_k_integral", "bessel_k_series", "fixed_window_log_bessel_k",
                 "log_integrand", "log_integrand_d1", "log_integrand_d2", "temme_pair"]
    for n in ref_names:
        assert n in bg.__all__ and hasattr(bg, n)
    spec_names = ["MaternParams", "LocationSet", "TileSpec", "CovarianceMatrix", "matern",
                  "generate_tile", "generate_covariance", "normalize_locations", "morton_order"]
    for n in spec_names:
        assert hasattr(bg, n)


def _msg(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        return f"{type(e).__name__}: {e}"
    return "<no error>"


def test_domain_errors_match_reference(golden):
    g = golden("api")
    ref = dict(zip(g["err_names"], g["err_msgs"]))
    cases = {
        "x0": lambda: bg.bessel_k(bg.EvalPoint(0.0, 1.0)),
        "xneg": lambda: bg.EvalPoint(-1.0, 1.0),
        "nunan": lambda: bg.EvalPoint(1.0, float("nan")),
        "series_big": lambda: bg.bessel_k_series(bg.EvalPoint(0.5, 1.0)),
        "integral_small": lambda: bg.bessel_k_integral(bg.EvalPoint(0.05, 1.0)),
        "temme_mu": lambda: bg.temme_pair(0.05, 0.5),
        "temme_x": lambda: bg.temme_pair(0.2, 0.0),
        "cfg_bins": lambda: bg.QuadratureConfig(bins=1),
        "cfg_t": lambda: bg.QuadratureConfig(t_lower=9.0, t_upper=9.0),
        "fw_x0": lambda: bg.fixed_window_log_bessel_k(0.0, 1.0),
    }
    for name, fn in cases.items():
        assert _msg(fn) == str(ref[name]), name


def test_config_and_result_types():
    c = bg.DEFAULT_CONFIG
    assert (c.t_lower, c.t_upper, c.bins, c.small_x_threshold, c.series_cap) == (0.0, 9.0, 40, 0.1, 15000)
    assert c.eps_machine == 2.0 ** -52
    with pytest.raises(bg.DomainError, match="small_x_threshold must be positive"):
        bg.QuadratureConfig(small_x_threshold=0.0)
    with pytest.raises(bg.DomainError, match="series_cap must be at least 1"):
        bg.QuadratureConfig(series_cap=0)
    r1 = bg.BesselResult(1.0, math.e, bg.PathTaken.INTEGRAL, warning="a")
    r2 = bg.BesselResult(1.0, math.e, bg.PathTaken.INTEGRAL, warning="b")
    assert r1 == r2  # warning excluded from equality, as in the reference
    cc = c.to_c(bins=16)
    assert cc.bins == 16 and cc.t_upper == 9.0


def test_result_overflow_and_warning():
    from paper_2502_00356_b200.besselk import _result

    p = bg.EvalPoint(1e-300, 30.0)
    r = _result(2e4, bg.PathTaken.SERIES, p)
    assert r.value == math.inf and "outside the validated region" in r.warning
    assert _result(0.0, bg.PathTaken.INTEGRAL, bg.EvalPoint(1.0, 1.0)).warning is None


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_numeric_calls_fail_loudly_without_gpu():
    with pytest.raises(bg.BackendUnavailable):
        bg.bessel_k(bg.EvalPoint(1.0, 1.0))
    with pytest.raises(bg.BackendUnavailable):
        bg.generate_covariance(np.random.default_rng(0).random((4, 2)), bg.MaternParams(1, 0.1, 1.5))
    with pytest.raises(bg.BackendUnavailable):
        bg.bessel_k_batch(np.ones(3), np.ones(3), validate=False)


def test_matern_params_and_locations():
    with pytest.raises(bg.DomainError, match="beta must be finite and positive"):
        bg.MaternParams(1.0, 0.0, 1.5)
    with pytest.raises(bg.DomainError, match="nu must be finite and positive"):
        bg.MaternParams(1.0, 0.1, float("inf"))
    with pytest.raises(bg.DomainError, match="duplicate"):
        bg.LocationSet(np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 0.0]]))
    with pytest.raises(bg.DomainError, match="shape"):
        bg.LocationSet(np.zeros((3, 3)))
    s = bg.LocationSet(np.array([[0.0, 0.0], [0.0, 0.0]]), reject_duplicates=False)
    assert len(s) == 2
    with pytest.raises(bg.DomainError):
        bg.TileSpec(0, 0, 1, 1, tile_size=0)
    with pytest.raises(bg.DomainError, match="r must be finite and nonnegative"):
        bg.matern(-1.0, bg.MaternParams(1, 1, 1))
    assert bg.matern(0.0, bg.MaternParams(2.5, 0.1, 1.5)) == 2.5  # r = 0 -> sigma^2, no GPU


def test_normalize_locations_spec_examples():
    """SPEC.md:293-296"""
    a = bg.normalize_locations(bg.LocationSet(np.array([[0.0, 0.0], [2.0, 1.0]])))
    assert np.array_equal(a.coords, [[0.0, 0.0], [1.0, 0.5]]) and a.normalized
    b = bg.normalize_locations(bg.LocationSet(np.array([[10.0, 10.0], [10.0, 12.0], [11.0, 10.0]])))
    assert np.array_equal(b.coords, [[0.0, 0.0], [0.0, 1.0], [0.5, 0.0]])
    u = np.array([[0.0, 0.0], [1.0, 1.0], [0.25, 0.75]])
    assert np.array_equal(bg.normalize_locations(bg.LocationSet(u)).coords, u)
    with pytest.raises(bg.DomainError, match="coincide"):
        bg.normalize_locations(bg.LocationSet(np.array([[1.0, 1.0]])))


def test_morton_order_spec_examples():
    """SPEC.md:302-305"""
    s = bg.LocationSet(np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 1.0], [1.0, 0.0]]), normalized=True)
    m, perm = bg.morton_order(s)
    assert np.array_equal(m.coords, [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    assert np.array_equal(s.coords[perm], m.coords) and m.ordering == bg.Ordering.MORTON
    one = bg.LocationSet(np.array([[0.3, 0.4]]), normalized=True)
    assert np.array_equal(bg.morton_order(one)[0].coords, one.coords)
    rng = np.random.default_rng(0)
    r = bg.LocationSet(rng.random((1000, 2)), normalized=True)
    mo, p = bg.morton_order(r)
    assert sorted(map(tuple, mo.coords)) == sorted(map(tuple, r.coords))

    def mean_step(c):
        return np.mean(np.linalg.norm(np.diff(c, axis=0), axis=1))

    assert mean_step(mo.coords) <= mean_step(r.coords)
    with pytest.raises(bg.DomainError, match="normalized"):
        bg.morton_order(bg.LocationSet(rng.random((5, 2))))


def test_cvmx_roundtrip_and_tile_accessors(tmp_path):
    rng = np.random.default_rng(1)
    a = rng.random((5, 5))
    a = a + a.T
    m = bg.CovarianceMatrix(N=5, data=a, tile_size=2)
    path = os.path.join(tmp_path, "m.cvmx")
    m.write_cvmx(path)
    raw = open(path, "rb").read()
    assert raw[:4] == b"CVMX" and len(raw) == 16 + 25 * 8
    back = bg.CovarianceMatrix.read_cvmx(path)
    assert np.array_equal(back.data, a)
    assert np.array_equal(m.tile(2, 1), a[4:5, 2:4])
    # packed lower tiles: tile l = p(p+1)/2 + q stored column-major
    ts, T = 2, 3
    packed = np.zeros((T * (T + 1) // 2, ts, ts))
    for p in range(T):
        for q in range(p + 1):
            blk = a[p * ts:(p + 1) * ts, q * ts:(q + 1) * ts]
            packed[p * (p + 1) // 2 + q][:blk.shape[1], :blk.shape[0]] = blk.T
    pm = bg.CovarianceMatrix(N=5, data=packed, layout="lower_tiles", tile_size=ts)
    for p in range(T):
        for q in range(T):
            assert np.array_equal(pm.tile(p, q), a[p * ts:(p + 1) * ts, q * ts:(q + 1) * ts])
    assert bg.lower_tile_count(5, 2) == 6


def test_morton_permutation_equivariance_host():
    """Entries are pure functions of location pairs, so any host reordering of the
    input permutes the matrix (checked bitwise on the GPU in the parity suite);
    here: the permutation returned by morton_order is a valid permutation."""
    rng = np.random.default_rng(5)
    s = bg.normalize_locations(bg.LocationSet(rng.random((257, 2)) * 7.0))
    m, perm = bg.morton_order(s, bits_per_axis=10)
    assert np.array_equal(np.sort(perm), np.arange(257))


def test_csv_roundtrip(tmp_path):
    rng = np.random.default_rng(2)
    a = rng.random((6, 6))
    a = a + a.T
    m = bg.CovarianceMatrix(N=6, data=a)
    path = os.path.join(tmp_path, "m.csv")
    m.write_csv(path)
    assert open(path).readline().count(",") == 5
    assert np.array_equal(bg.CovarianceMatrix.read_csv(path).data, a)
