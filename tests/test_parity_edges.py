"""Edge-case GPU parity for the Matern kernel against the CPU oracle: extreme
sigma^2 (exp range fallback), tiny / huge range beta (underflow, last LUT bucket,
all-series), small and large nu, large coordinates, tile-edge sizes, unaligned
row blocks and non-default quadrature configs."""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def bg():
    import paper_2502_00356_b200 as bg

    return bg


def _cmp(bg, oracle, locs, s2, beta, nu, cfg=None, rows=None):
    cfg = cfg or bg.DEFAULT_CONFIG
    theta = bg.MaternParams(s2, beta, nu)
    got = bg.generate_covariance(locs, theta, cfg, device="cuda", rows=rows).to_numpy()
    ref = oracle.generate_covariance(locs, s2, beta, nu, t0=cfg.t_lower, t1=cfg.t_upper,
                                     bins=cfg.bins, thr=cfg.small_x_threshold,
                                     series_cap=cfg.series_cap, threads=8, row_range=rows)
    both_zero = (got == 0.0) & (ref == 0.0)
    err = rel_err(got, ref)
    err[both_zero] = 0.0
    # entries the reference rounds into the subnormal range carry absolute error only
    tiny = np.abs(ref) < 1e-290
    assert np.max(np.where(tiny, 0.0, err)) <= TOL, (s2, beta, nu)
    assert np.max(np.abs(got - ref)[tiny], initial=0.0) <= 1e-300
    return got


@pytest.mark.parametrize("s2", [1e-300, 1e-30, 1.0, 1e30, 1e300])
def test_extreme_variance(bg, oracle, s2):
    locs = np.random.default_rng(1).random((150, 2))
    _cmp(bg, oracle, locs, s2, 0.1, 1.5)


@pytest.mark.parametrize("beta", [1e-4, 0.003, 0.1, 5.0, 1e4])
def test_range_extremes(bg, oracle, beta):
    locs = np.random.default_rng(2).random((180, 2))
    _cmp(bg, oracle, locs, 1.0, beta, 0.8)


@pytest.mark.parametrize("nu", [1e-3, 0.05, 0.5, 1.0, 2.0, 7.5, 19.99, 25.0, 40.0])
def test_smoothness_range(bg, oracle, nu):
    locs = np.random.default_rng(3).random((160, 2))
    _cmp(bg, oracle, locs, 1.0, 0.1, nu)


def test_large_coordinates(bg, oracle):
    locs = np.random.default_rng(4).random((200, 2)) * 1e6 + 3e7
    _cmp(bg, oracle, locs, 2.0, 1e5, 1.7)


@pytest.mark.parametrize("N", [1, 2, 63, 64, 65, 127, 129])
def test_tile_edge_sizes(bg, oracle, N):
    locs = np.random.default_rng(5 + N).random((N, 2))
    got = _cmp(bg, oracle, locs, 1.0, 0.1, 1.5)
    assert np.array_equal(got, got.T)


@pytest.mark.parametrize("rows", [(0, 1), (63, 64), (64, 129), (1, 130), (100, 131)])
def test_unaligned_row_blocks(bg, oracle, rows):
    locs = np.random.default_rng(6).random((131, 2))
    _cmp(bg, oracle, locs, 1.0, 0.1, 2.9, rows=rows)


@pytest.mark.parametrize("kw", [dict(t_lower=0.5, t_upper=7.0), dict(bins=7), dict(bins=200),
                                dict(series_cap=1), dict(small_x_threshold=1e-3),
                                dict(small_x_threshold=2.0)])
def test_nondefault_configs(bg, oracle, kw):
    locs = np.random.default_rng(7).random((140, 2))
    locs[3] = locs[2] + 1e-4  # a series entry
    _cmp(bg, oracle, locs, 1.0, 0.1, 1.3, cfg=bg.QuadratureConfig(**kw))
