"""Accuracy audit on the GPU: the reference's oracle.py surface.

The reference audits its production path against a dynamic-window Takekawa
integrator with 2^16 bins (oracle.py:92-160) and reports the paper's RE metric
as heatmaps (oracle.py:162-262); its bound finder (Algorithm 1)
sweeps candidate upper bounds with the same machinery.  In the reference these
run one point at a time in Python/numba (minutes to hours); here every grid is
one launch of ``bgk_log_grid`` (one CTA per point, reference-faithful window
search and node arithmetic) or of the BesselK batch kernel.

    oracle_log_bessel_k, oracle_log10_grid, refined_log10_grid,
    pure_integral_log10_grid, relative_error, RelErrorGrid, error_heatmap,
    find_upper_bound
"""

from __future__ import annotations

import ctypes
import io
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .besselk import (DEFAULT_CONFIG, EPS_MACHINE, DomainError, EvalPoint, QuadratureConfig,
                      bessel_k_batch)

DEFAULT_ORACLE_BINS = 2 ** 16  # oracle.py:28
METHODS = ("refined", "pure-integral", "oracle-vs-oracle")  # oracle.py:220


class ConvergenceError(RuntimeError):  # oracle.py:34-35
    """A root finder failed to bracket or converge."""


def _log_grid(nus, xs, cfg: QuadratureConfig, method: int, bins: int, base10: bool) -> np.ndarray:
    import torch

    L = _lib.lib()
    nus = np.ascontiguousarray(nus, dtype=np.float64).ravel()
    xs = np.ascontiguousarray(xs, dtype=np.float64).ravel()
    nd = torch.from_numpy(nus).cuda()
    xd = torch.from_numpy(xs).cuda()
    out = torch.empty((nus.size, xs.size), dtype=torch.float64, device="cuda")
    c = cfg.to_c()
    _lib.check(L.bgk_log_grid(nd.data_ptr(), nus.size, xd.data_ptr(), xs.size, ctypes.byref(c),
                              method, int(bins), 1 if base10 else 0, out.data_ptr(),
                              torch.cuda.current_stream().cuda_stream), "bgk_log_grid")
    return out.cpu().numpy()


def oracle_log_bessel_k(p: EvalPoint, bins: int = DEFAULT_ORACLE_BINS,
                        cfg: QuadratureConfig = DEFAULT_CONFIG) -> float:
    """Reference log K (oracle.py:137-151): the series below the threshold, else the
    dynamic-window quadrature with ``bins`` intervals."""
    if p.x <= 0.0:
        raise DomainError("x must be positive")
    if bins < 1:
        raise DomainError("bins must be positive")
    v = float(_log_grid([p.nu], [p.x], cfg, _lib_method("oracle"), bins, False)[0, 0])
    if not math.isfinite(v):
        raise ConvergenceError(f"window search failed at (x={p.x!r}, nu={p.nu!r})")
    return v


def _lib_method(name: str) -> int:
    return {"refined": 0, "pure-integral": 1, "oracle": 2}[name]


def oracle_log10_grid(nus, xs, bins: int = DEFAULT_ORACLE_BINS,
                      cfg: QuadratureConfig = DEFAULT_CONFIG, workers: int = 1) -> np.ndarray:
    """Reference base-10 log K over a (nu, x) grid (oracle.py:194-217); NaN where the
    window search fails.  ``workers`` is accepted for API compatibility."""
    return _log_grid(nus, xs, cfg, _lib_method("oracle"), bins, True)


def refined_log10_grid(nus, xs, cfg: QuadratureConfig = DEFAULT_CONFIG) -> np.ndarray:
    """Production evaluator, base 10 (kernels.py:306-318)."""
    return _log_grid(nus, xs, cfg, _lib_method("refined"), cfg.bins, True)


def pure_integral_log10_grid(nus, xs, cfg: QuadratureConfig = DEFAULT_CONFIG) -> np.ndarray:
    """Fixed-window quadrature everywhere, also below the threshold (kernels.py:321-329)."""
    return _log_grid(nus, xs, cfg, _lib_method("pure-integral"), cfg.bins, True)


def relative_error(reference: float, output: float) -> float:
    """RE = log10(1 + |reference - output| / eps_machine) (oracle.py:162-167)."""
    if not (math.isfinite(reference) and math.isfinite(output)):
        raise DomainError("relative_error needs finite inputs")
    return math.log10(1.0 + abs(reference - output) / EPS_MACHINE)


@dataclass(frozen=True)
class RelErrorGrid:  # oracle.py:170-191
    """RE per (nu, x) cell; invalid cells are NaN and excluded from max_re."""

    nus: np.ndarray
    xs: np.ndarray
    re: np.ndarray
    method: str

    @property
    def max_re(self) -> float:
        return float(np.nanmax(self.re))

    def to_csv(self, path_or_buf) -> None:
        buf = path_or_buf if hasattr(path_or_buf, "write") else io.StringIO()
        buf.write("nu,x,re\n")
        for i, nu in enumerate(self.nus):
            for j, x in enumerate(self.xs):
                buf.write(f"{nu:.17g},{x:.17g},{self.re[i, j]:.17g}\n")
        if buf is not path_or_buf:
            with open(path_or_buf, "w") as fh:
                fh.write(buf.getvalue())


def error_heatmap(grid_nu, grid_x, method: str, cfg: QuadratureConfig = DEFAULT_CONFIG,
                  oracle_bins: int = DEFAULT_ORACLE_BINS, reference=None,
                  workers: int = 1) -> RelErrorGrid:
    """RE of a method against the oracle over a (nu, x) grid (oracle.py:223-262)."""
    nus = np.asarray(grid_nu, dtype=np.float64)
    xs = np.asarray(grid_x, dtype=np.float64)
    if nus.size == 0 or xs.size == 0:
        raise DomainError("grids must be non-empty")
    if np.any(xs <= 0.0):
        raise DomainError("x grid must be positive")
    if method not in METHODS:
        raise DomainError(f"method must be one of {METHODS}")
    if reference is None:
        reference = oracle_log10_grid(nus, xs, bins=oracle_bins, cfg=cfg)
    reference = np.asarray(reference, dtype=np.float64)
    if reference.shape != (nus.size, xs.size):
        raise DomainError("reference grid shape mismatch")
    if method == "refined":
        out = refined_log10_grid(nus, xs, cfg)
    elif method == "pure-integral":
        out = pure_integral_log10_grid(nus, xs, cfg)
    else:
        out = oracle_log10_grid(nus, xs, bins=cfg.bins, cfg=cfg)
    with np.errstate(invalid="ignore"):
        re = np.log10(1.0 + np.abs(reference - out) / EPS_MACHINE)
    re[~np.isfinite(out) | ~np.isfinite(reference)] = np.nan
    return RelErrorGrid(nus=nus, xs=xs, re=re, method=method)


class NoBoundFound(RuntimeError):
    """No candidate upper bound meets the tolerance."""


def bound_region_grid(thr: float = 0.1):
    """141 x 40 linear grid (x = 0 replaced by the threshold) plus 50
    log-spaced x in [0.1, 1]; nu in (0, 20]."""
    xs = np.linspace(0.0, 140.0, 141)
    xs[0] = thr
    xs = np.unique(np.concatenate([xs, np.geomspace(0.1, 1.0, 50)]))
    nus = np.linspace(0.5, 20.0, 40)
    return nus, xs


def find_upper_bound(candidates=(5, 6, 7, 8, 9, 10, 11, 12), tol: float = 1e-9,
                     bins: int = 2 ** 12, region=None, cfg: QuadratureConfig = DEFAULT_CONFIG,
                     return_curve: bool = False):
    """Algorithm 1: smallest L with max |oracle_log -
    fixed_window_log([0, L], bins)| <= tol over the region grid (natural logs)."""
    nus, xs = region if region is not None else bound_region_grid(cfg.small_x_threshold)
    ref = _log_grid(nus, xs, cfg, _lib_method("oracle"), bins, False)
    NU, X = np.meshgrid(nus, xs, indexing="ij")
    curve = []
    found = None
    for L in candidates:
        c = QuadratureConfig(t_lower=0.0, t_upper=float(L), bins=bins,
                             small_x_threshold=cfg.small_x_threshold,
                             series_cap=cfg.series_cap, eps_machine=cfg.eps_machine)
        fw = bessel_k_batch(X.ravel(), NU.ravel(), c, route="integral",
                            validate=False).log_value.reshape(NU.shape)
        ae = float(np.nanmax(np.abs(ref - fw)))
        curve.append((float(L), ae))
        if found is None and ae <= tol:
            found = float(L)
    if return_curve:
        return found, curve
    if found is None:
        raise NoBoundFound(f"no candidate meets {tol:g}: {curve}")
    return found
