"""TEST / MEASUREMENT INFRASTRUCTURE ONLY -- the reference package itself on the CPU.

Drives the UNMODIFIED reference numba kernels (``besselgp.kernels`` from
``baseline/_ref``, installed with ``pip install --no-index --no-deps --target
baseline/_ref`` from a copy of /root/reference/pkg) the way the
reference's own code and SPEC call them:

* BesselK batch: a numba ``@njit(nogil)`` loop over ``kernels.refined_log_bessel``
  (kernels.py:296-302) run in chunks on a ThreadPoolExecutor -- the reference's
  threading idiom (oracle.py:211-213).
* Matern: the caller the reference only specifies (restated:
  h = (t1 - t0)/b, c_m = cosh(t0 + m h), a_m = kernels.log_cosh(nu t_m),
  lp = log(sigma2) - (nu - 1) ln2 - lgamma(nu), kernels.py:343-345) -- lower
  tiles through ``kernels.matern_tile`` (kernels.py:338-381) on the thread pool,
  each off-diagonal tile mirrored into the upper triangle.

Only bench.py's ``--impl reference`` / CPU-baseline legs use this module, as the
timed CPU reference -- never the product path.  It needs numba and the installed
reference; ``available()`` says whether both are present.
"""

from __future__ import annotations

import math
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(_ROOT, "baseline", "_ref")
LN2 = 0.6931471805599453

_K = None
_err = None


def kernels():
    """The reference's ``besselgp.kernels`` module (imported once) or None."""
    global _K, _err
    if _K is None and _err is None:
        try:
            os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench_ref")
            if REF_DIR not in sys.path:
                sys.path.insert(0, REF_DIR)
            import besselgp.kernels as K  # noqa: PLC0415

            if not os.path.realpath(K.__file__).startswith(os.path.realpath(REF_DIR)):
                raise ImportError(f"besselgp resolved to {K.__file__}, not baseline/_ref")
            _K = K
        except Exception as e:  # noqa: BLE001
            _err = f"{type(e).__name__}: {e}"
    return _K


def available() -> bool:
    return kernels() is not None


def unavailable_reason() -> str | None:
    kernels()
    return _err


_bk_loop = None


def _bk_loop_fn():
    global _bk_loop
    if _bk_loop is None:
        from numba import njit  # noqa: PLC0415

        refined = kernels().refined_log_bessel

        @njit(nogil=True)
        def loop(x, nu, out, t0, t1, bins, thr, eps, cap):
            for i in range(x.shape[0]):
                out[i] = refined(x[i], nu[i], t0, t1, bins, thr, eps, cap)

        _bk_loop = loop
    return _bk_loop


def refined_log_bessel_batch(x, nu, threads, t0=0.0, t1=9.0, bins=40, thr=0.1,
                             eps=2.0 ** -52, cap=15000, chunks=256) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    nu = np.ascontiguousarray(nu, dtype=np.float64)
    out = np.empty_like(x)
    loop = _bk_loop_fn()
    edges = np.linspace(0, x.size, min(chunks, max(1, x.size)) + 1).astype(np.int64)

    def run(i):
        a, b = edges[i], edges[i + 1]
        loop(x[a:b], nu[a:b], out[a:b], t0, t1, bins, thr, eps, cap)

    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(run, range(len(edges) - 1)))
    return out


def matern_caller_tables(sigma_sq, nu, t0=0.0, t1=9.0, bins=40):
    """The restated caller's per-call tables (kernels.py:343-345)."""
    K = kernels()
    h = (t1 - t0) / bins
    c = np.empty(bins + 1)
    a = np.empty(bins + 1)
    for m in range(bins + 1):
        t = t0 + m * h
        c[m] = math.cosh(t)
        a[m] = K.log_cosh(nu * t)
    lp = math.log(sigma_sq) - (nu - 1.0) * LN2 - math.lgamma(nu)
    return c, a, h, lp


def tri_index(l: int):
    p = int((math.sqrt(8.0 * l + 1.0) - 1.0) / 2.0)
    while (p + 1) * (p + 2) // 2 <= l:
        p += 1
    while p * (p + 1) // 2 > l:
        p -= 1
    return p, l - p * (p + 1) // 2


class CovarianceJob:
    """Restated generate_covariance of the full N x N matrix,
    runnable in slices of the lower-tile index range so one job can be spread
    over several timed steps: ``run(l0, l1)`` computes lower tiles [l0, l1) with
    kernels.matern_tile and mirrors each off-diagonal tile."""

    def __init__(self, locs, sigma_sq, beta, nu, out, threads, tile_size=256, t0=0.0,
                 t1=9.0, bins=40, thr=0.1, eps=2.0 ** -52, cap=15000):
        self.K = kernels()
        self.lx = np.ascontiguousarray(locs[:, 0], dtype=np.float64)
        self.ly = np.ascontiguousarray(locs[:, 1], dtype=np.float64)
        self.N = locs.shape[0]
        self.ts = tile_size
        self.T = -(-self.N // tile_size)
        self.ntiles = self.T * (self.T + 1) // 2
        self.out = out
        self.threads = threads
        self.c, self.a, self.h, self.lp = matern_caller_tables(sigma_sq, nu, t0, t1, bins)
        self.args = (sigma_sq, beta, nu, self.lp)
        self.cfg = (thr, eps, cap)
        self.pool = ThreadPoolExecutor(max_workers=threads)

    def _tile(self, l):
        p, q = tri_index(l)
        ts, N = self.ts, self.N
        r0, c0 = p * ts, q * ts
        m, n = min(ts, N - r0), min(ts, N - c0)
        blk = self.out[r0:r0 + m, c0:c0 + n]
        self.K.matern_tile(blk, self.lx[r0:r0 + m], self.ly[r0:r0 + m], self.lx[c0:c0 + n],
                           self.ly[c0:c0 + n], *self.args, self.c, self.a, self.h, *self.cfg)
        if p != q:
            self.out[c0:c0 + n, r0:r0 + m] = blk.T

    def run(self, l0: int, l1: int):
        # chunks of consecutive tiles per task (fewer executor round trips)
        step = 8
        list(self.pool.map(lambda s: [self._tile(l) for l in range(s, min(l1, s + step))],
                           range(l0, l1, step)))

    def close(self):
        self.pool.shutdown()
