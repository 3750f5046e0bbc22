"""Coverage of the BesselK fast path's node windows (bgk_besselk.cu: the host-built
(x, nu)-cell table of extents above/below the anchor node).

For a dense sample of every table cell (edges included, far denser than the 5 x 5
sample the table is built from) every node the reference keeps -- g_k - g_max >
-33 with g the log-integrand on the grid and g_max its grid maximum
(kernels.py:112-123, 154-209; the reference walks to -46, the nodes in (-46, -33]
add < 41 e^-33 = 1.9e-13 of the sum, far inside the 1e-10 parity tolerance) -- must lie inside the window [lo, hi] the
kernel sums.  The CPU test uses the host anchor (fp32 asinhf); the GPU test the
kernel's own classify pass and fast fp32 anchor (bgk_besselk_windows).
"""

import ctypes

import numpy as np
import pytest

import paper_2502_00356_b200 as bg
from paper_2502_00356_b200 import _lib

CUT = 33.0  # bgk_besselk.cu: BGK_BK_WCUT - 1
X_BITS = 2          # BGK_BK_XBITS: 4 x cells per octave, 16 octaves from 2^-6
NU_STEP = 2         # BGK_BK_NUSTEP: nu cells of width 1/2, 24 units


def _log_cosh(z):
    z = np.abs(z)
    with np.errstate(over="ignore"):
        small = np.log(np.cosh(np.minimum(z, 25.0)))
    big = z - np.log(2.0) + np.log1p(np.exp(-2.0 * z))
    return np.where(z < 25.0, small, big)


def reference_windows(x, nu, cfg):
    """Per point: (first grid argmax, lowest and highest node with g - g_max > -CUT)."""
    b = cfg.bins
    h = (cfg.t_upper - cfg.t_lower) / b
    t = cfg.t_lower + np.arange(b + 1) * h
    g = _log_cosh(np.abs(nu)[:, None] * t[None, :]) - x[:, None] * np.cosh(t)[None, :]
    ms = np.argmax(g, axis=1)
    keep = g - g[np.arange(len(x)), ms][:, None] > -CUT
    k = np.arange(b + 1)
    lo = np.where(keep, k[None, :], b + 1).min(axis=1)
    hi = np.where(keep, k[None, :], -1).max(axis=1)
    return ms, lo, hi


def dense_cell_samples(per_axis=12, nu_max=24.0):
    """Every (x, nu) cell of the table, per_axis^2 points each, edges included."""
    xs, ns = [], []
    f = np.linspace(0.0, 1.0, per_axis)
    for key in range(16 << X_BITS):
        e, sub = divmod(key, 1 << X_BITS)
        lo = 2.0 ** (e - 6) * (1 + sub / (1 << X_BITS))
        hi = 2.0 ** (e - 6) * (1 + (sub + 1) / (1 << X_BITS))
        xv = lo + (hi - lo) * f
        xv[-1] = np.nextafter(hi, 0.0)
        for ci in range(int(nu_max * NU_STEP) - 1):
            nlo, nhi = ci / NU_STEP, (ci + 1) / NU_STEP
            nv = nlo + (nhi - nlo) * f
            nv[-1] = np.nextafter(nhi, 0.0)
            X, Nn = np.meshgrid(xv, nv)
            xs.append(X.ravel())
            ns.append(Nn.ravel())
    return np.concatenate(xs), np.concatenate(ns)


def _cfgs():
    return [bg.DEFAULT_CONFIG,
            bg.QuadratureConfig(t_lower=0.0, t_upper=12.0, bins=96, small_x_threshold=0.05),
            bg.QuadratureConfig(bins=16)]


def _check(x, nu, m, lo, hi, cfg):
    fast = m >= 0
    assert fast.mean() > 0.5  # most of the sample takes the windowed fast path
    ms, rlo, rhi = reference_windows(x[fast], nu[fast], cfg)
    bad = (rlo < lo[fast]) | (rhi > hi[fast])
    if bad.any():
        i = np.flatnonzero(bad)[:5]
        pytest.fail(f"{bad.sum()} of {fast.sum()} windows miss reference nodes, e.g. "
                    f"x={x[fast][i]} nu={nu[fast][i]} ours=[{lo[fast][i]}, {hi[fast][i]}] "
                    f"ref=[{rlo[i]}, {rhi[i]}] (argmax {ms[i]}, anchor {m[fast][i]})")


@pytest.mark.parametrize("ci", range(3))
def test_window_table_covers_reference_windows_host_anchor(ci):
    cfg = _cfgs()[ci]
    x0, nu0 = dense_cell_samples()
    keep = x0 >= cfg.small_x_threshold
    x, nu = x0[keep], nu0[keep]
    n = len(x)
    m = np.empty(n, np.int32)
    lo = np.empty(n, np.int32)
    hi = np.empty(n, np.int32)
    c = cfg.to_c()
    L = _lib.load_library()
    _lib.check(L.bgk_besselk_windows_host(x.ctypes.data, nu.ctypes.data, n, ctypes.byref(c),
                                          m.ctypes.data, lo.ctypes.data, hi.ctypes.data),
               "bgk_besselk_windows_host")
    _check(x, nu, m, lo, hi, cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(3))
def test_window_table_covers_reference_windows_device_anchor(ci):
    import torch

    cfg = _cfgs()[ci]
    x0, nu0 = dense_cell_samples()
    keep = x0 >= cfg.small_x_threshold
    x, nu = x0[keep], nu0[keep]
    rng = np.random.default_rng(11)  # plus the BK distribution
    xr = 140.0 * (1.0 - rng.random(200_000))
    nr = 20.0 * (1.0 - rng.random(200_000))
    keep = xr >= cfg.small_x_threshold
    x = np.concatenate([x, xr[keep]])
    nu = np.concatenate([nu, nr[keep]])
    n = len(x)
    xd = torch.from_numpy(x).cuda()
    nd = torch.from_numpy(nu).cuda()
    m = torch.empty(n, dtype=torch.int32, device="cuda")
    lo = torch.empty_like(m)
    hi = torch.empty_like(m)
    c = cfg.to_c()
    _lib.check(_lib.lib().bgk_besselk_windows(xd.data_ptr(), nd.data_ptr(), n, ctypes.byref(c),
                                              m.data_ptr(), lo.data_ptr(), hi.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream),
               "bgk_besselk_windows")
    _check(x, nu, m.cpu().numpy(), lo.cpu().numpy(), hi.cpu().numpy(), cfg)
