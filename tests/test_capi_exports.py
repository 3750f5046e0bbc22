"""CPU checks of the C-ABI boundary: the library loads without a GPU, exports every
symbol include/besselgp_b200.h declares, validates arguments before touching
CUDA, and builds correct host-side Matern plans (node tables, LUT windows)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "besselgp_b200.h")


@pytest.fixture(scope="module")
def L():
    from paper_2502_00356_b200 import _lib

    return _lib.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bgk_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound(L):
    from paper_2502_00356_b200 import _lib

    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n  # dlsym succeeds
        assert n in _lib.SIGNATURES, f"{n} has no ctypes binding"


def test_abi_and_struct_layout(L):
    from paper_2502_00356_b200 import _lib

    assert L.bgk_abi_version() == _lib.BGK_ABI_VERSION
    assert L.bgk_matern_plan_size() == ctypes.sizeof(_lib.BgkMaternPlan)
    assert ctypes.sizeof(_lib.BgkConfig) == 48


def test_argument_validation_without_gpu(L):
    """Bad arguments are rejected before any CUDA call (safe on a CPU box)."""
    from paper_2502_00356_b200 import _lib

    cfg = _lib.BgkConfig(0.0, 9.0, 40, 0.1, 15000, 2.0 ** -52)
    bad_cfg = _lib.BgkConfig(9.0, 9.0, 40, 0.1, 15000, 2.0 ** -52)
    assert L.bgk_besselk_batch(None, None, -1, ctypes.byref(cfg), 0, None, None, None, None) == -1
    assert L.bgk_besselk_batch(None, None, 5, ctypes.byref(cfg), 0, None, None, None, None) == -1
    assert L.bgk_besselk_batch(None, None, 0, ctypes.byref(bad_cfg), 0, None, None, None, None) == -1
    assert b"invalid bgk_config" in L.bgk_last_error()
    assert L.bgk_besselk_batch(None, None, 0, ctypes.byref(cfg), 7, None, None, None, None) == -1
    assert L.bgk_log_integrand_batch(None, None, None, 1, 3, None, None) == -1
    # the scalar entry point: config, route and result pointer checked first
    out = ctypes.c_double()
    assert L.bgk_besselk_scalar(1.0, 1.5, None, 0, ctypes.byref(out), None) == -1
    assert L.bgk_besselk_scalar(1.0, 1.5, ctypes.byref(cfg), 3, ctypes.byref(out), None) == -1
    assert L.bgk_besselk_scalar(1.0, 1.5, ctypes.byref(bad_cfg), 0, ctypes.byref(out), None) == -1
    assert L.bgk_besselk_scalar(1.0, 1.5, ctypes.byref(cfg), 0, None, None) == -1
    assert b"bgk_besselk_scalar" in L.bgk_last_error()
    plan = _lib.BgkMaternPlan()
    assert L.bgk_matern_tile(ctypes.byref(plan), None, None, 1, None, None, 1, None, 1, 0, None) == -1
    assert b"uninitialised" in L.bgk_last_error()
    assert L.bgk_matern_plan_init(ctypes.byref(plan), 1.0, 0.1, 1.5, ctypes.byref(cfg)) == 0
    assert L.bgk_matern_covariance(ctypes.byref(plan), None, None, 10, 5, 3, None, 10, 0, None) == -1
    assert L.bgk_matern_lower_tiles(ctypes.byref(plan), None, None, 10, 0, 0, 1, None, None) == -1
    # empty work is a no-op success (no launch)
    assert L.bgk_matern_tile(ctypes.byref(plan), None, None, 0, None, None, 5, None, 5, 0, None) == 0
    big = _lib.BgkConfig(0.0, 9.0, 5000, 0.1, 15000, 2.0 ** -52)
    assert L.bgk_matern_plan_init(ctypes.byref(plan), 1.0, 0.1, 1.5, ctypes.byref(cfg)) == 0
    # multi-GPU peer entry points: owners / rank / ranges checked before any launch
    N, G = 1000, 2
    T = -(-N // 64)
    starts = (ctypes.c_int64 * 3)(0, 8, T)
    bases = (ctypes.c_void_p * 2)(1, 2)
    assert L.bgk_matern_covariance_peer_band(ctypes.byref(plan), None, None, N, G, starts, bases,
                                             2, None) == -1  # rank outside [0, G)
    assert b"rank" in L.bgk_last_error()
    bad = (ctypes.c_int64 * 3)(0, 8, T + 1)
    assert L.bgk_matern_covariance_peer_band(ctypes.byref(plan), None, None, N, G, bad, bases,
                                             0, None) == -1
    assert L.bgk_matern_covariance_peer(ctypes.byref(plan), None, None, N, G, starts, bases, 0,
                                        T * (T + 1) // 2 + 1, None) == -1  # tile range
    assert L.bgk_matern_covariance_peer(ctypes.byref(plan), None, None, N, G, starts, bases, 0,
                                        0, None) == 0  # empty range: no-op
    assert L.bgk_matern_plan_init(ctypes.byref(plan), 1.0, 0.1, 1.5, ctypes.byref(big)) == -3


def _plan(nu, cfg=None, sigma_sq=1.0, beta=0.1):
    import paper_2502_00356_b200 as bg

    return bg.matern_plan(bg.MaternParams(sigma_sq, beta, nu), cfg or bg.DEFAULT_CONFIG)


@pytest.mark.parametrize("nu", [0.3, 0.8, 1.5, 1.7, 2.9, 5.3, 19.5])
def test_plan_tables_match_oracle_caller(oracle, nu):
    p = _plan(nu)
    c, a, h = oracle.matern_tables(nu)
    assert p.nnodes == 41 and p.h == h
    assert np.array_equal(np.array(p.c[:41]), c)
    assert np.array_equal(np.array(p.a[:41]), a)
    assert p.log_prefactor == oracle.matern_log_prefactor(1.0, nu)
    assert p.m_steps == math.floor(nu + 0.5)


def _key(u, shift):
    return int(np.array([u]).view(np.uint64)[0] >> np.uint64(32 + shift))


@pytest.mark.parametrize("nu,bins", [(0.3, 40), (1.5, 40), (2.9, 40), (19.5, 40), (1.5, 16),
                                     (1.5, 128), (0.8, 7)])
def test_lut_windows_cover_reference_windows(nu, bins):
    """For u across the whole LUT range, every node with dg > -33 from the grid
    argmax lies in the bucket's [lo, hi]: the reference keeps dg > -46
    (kernels.py:363-379), so the nodes it sums that the kernel drops add up to
    < 41 e^-33 = 1.9e-13 of the peak term (BGK_WINDOW_CUTOFF; inside the 1e-10 tolerance).  And
    y = g_k - g_anchor stays inside the table exp's range."""
    import paper_2502_00356_b200 as bg

    cfg = bg.QuadratureConfig(bins=bins)
    p = _plan(nu, cfg)
    assert p.fast == 1
    nn = p.nnodes
    c = np.array(p.c[:nn])
    a = np.array(p.a[:nn])
    rng = np.random.default_rng(1)
    us = np.concatenate([np.geomspace(0.1, 1e5, 4000), 0.1 + rng.random(500),
                         [0.1, np.nextafter(0.1, 1)]])
    lut = np.array(p.lut[:p.nbuckets])
    for u in us:
        g = a - u * c
        ms = int(np.argmax(g))
        keep = np.nonzero(g - g[ms] > -33.0)[0]
        b = min(max(_key(u, p.key_shift) - p.key_base, 0), p.nbuckets - 1)
        w = int(lut[b])
        anc, lo, hi = w & 1023, (w >> 10) & 1023, w >> 20
        assert lo <= keep.min() and keep.max() <= hi, (u, lo, hi, keep)
        assert p.anchor_min <= anc <= p.anchor_max
        y = g[lo:hi + 1] - g[anc]
        assert np.all(y < 30.0) and np.all(y > -700.0)
    # windows non-increasing in u (the kernel reads warp bounds from end lanes)
    lo_s = (lut >> 10) & 1023
    hi_s = lut >> 20
    assert np.all(np.diff(lo_s.astype(int)) <= 0) and np.all(np.diff(hi_s.astype(int)) <= 0)


def test_plan_from_reference_argument_list(oracle):
    """bgk_matern_plan_init_tables takes kernels.matern_tile's exact arguments."""
    from paper_2502_00356_b200 import _lib

    L = _lib.load_library()
    c, a, h = oracle.matern_tables(1.7)
    plan = _lib.BgkMaternPlan()
    rc = L.bgk_matern_plan_init_tables(ctypes.byref(plan), 2.0, 0.1, 1.7, 0.123,
                                       c.ctypes.data, a.ctypes.data, c.size, h, 0.1,
                                       2.0 ** -52, 15000)
    assert rc == 0 and plan.fast == 1 and plan.log_prefactor == 0.123
    assert plan.aw[0] == a[0] - 0.6931471805599453 and plan.aw[5] == a[5]
