"""Modified Bessel function of the second kind -- B200 build of besselk.py.

Same public names, dataclasses, validation, messages and routing as the
reference module (/root/reference/pkg/src/besselgp/besselk.py:1-165); the
numeric work that the reference hands to numba (kernels.py) runs in the sm_100a
kernels of libbesselgp_sm100a.so instead.  Small arguments (x below the
threshold, default 0.1) use the Temme series with a log-space forward
recurrence; everything else uses the fixed-window trapezoid log-sum-exp
quadrature over [t_lower, t_upper] with ``bins`` intervals.

Added for the GPU: ``bessel_k_batch`` (arrays / CUDA tensors in, arrays /
CUDA tensors out), the natural unit of work for a device.
"""

from __future__ import annotations

import ctypes
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _lib

EPS_MACHINE = 2.0 ** -52  # kernels.py:15

VALIDATED_X_MAX = 140.0  # besselk.py:19
VALIDATED_NU_MAX = 20.0  # besselk.py:20


class PathTaken(enum.Enum):  # besselk.py:23-25
    SERIES = "series"
    INTEGRAL = "integral"


class DomainError(ValueError):  # besselk.py:28-29
    """Input outside an operation's domain."""


@dataclass(frozen=True)
class QuadratureConfig:  # besselk.py:32-51
    """Operating point of the fixed-window quadrature and series."""

    t_lower: float = 0.0
    t_upper: float = 9.0
    bins: int = 40
    small_x_threshold: float = 0.1
    series_cap: int = 15000
    eps_machine: float = EPS_MACHINE

    def __post_init__(self):
        if not self.t_lower < self.t_upper:
            raise DomainError("t_lower must be below t_upper")
        if self.bins < 2:
            raise DomainError("bins must be at least 2")
        if self.small_x_threshold <= 0:
            raise DomainError("small_x_threshold must be positive")
        if self.series_cap < 1:
            raise DomainError("series_cap must be at least 1")

    def to_c(self, bins: int | None = None) -> _lib.BgkConfig:
        return _lib.BgkConfig(float(self.t_lower), float(self.t_upper),
                              int(self.bins if bins is None else bins),
                              float(self.small_x_threshold), int(self.series_cap),
                              float(self.eps_machine))


DEFAULT_CONFIG = QuadratureConfig()


@dataclass(frozen=True)
class EvalPoint:  # besselk.py:57-69
    """One (x, nu) evaluation point; negative orders fold via K_{-nu} = K_nu
    before construction."""

    x: float
    nu: float

    def __post_init__(self):
        if not (math.isfinite(self.x) and self.x >= 0.0):
            raise DomainError(f"x must be finite and nonnegative, got {self.x!r}")
        if not (math.isfinite(self.nu) and self.nu >= 0.0):
            raise DomainError(f"nu must be finite and nonnegative, got {self.nu!r}")


@dataclass(frozen=True)
class BesselResult:  # besselk.py:72-77
    log_value: float
    value: float
    path_taken: PathTaken
    warning: str | None = field(default=None, compare=False)


def _result(log_value: float, path: PathTaken, p: EvalPoint) -> BesselResult:  # besselk.py:80-91
    try:
        value = math.exp(log_value)
    except OverflowError:
        value = math.inf
    warning = None
    if p.x > VALIDATED_X_MAX or p.nu > VALIDATED_NU_MAX:
        warning = (
            f"(x={p.x:g}, nu={p.nu:g}) lies outside the validated region "
            f"[0, {VALIDATED_X_MAX:g}] x (0, {VALIDATED_NU_MAX:g}]"
        )
    return BesselResult(log_value, value, path, warning)


# ---------------------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------------------

def _torch():
    import torch

    return torch


def _stream_handle():
    """The current torch stream of the current device as a raw cudaStream_t (the
    C-level accessor when torch has it: ~10x cheaper than building a Stream object,
    which matters for the scalar API)."""
    torch = _torch()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(torch._C._cuda_getDevice())
    return torch.cuda.current_stream().cuda_stream


def _to_device(a, device=None):
    """float64 contiguous CUDA tensor view/copy of ``a`` (numpy, list, scalar or tensor)."""
    _lib.lib()  # BackendUnavailable (not a CPU fallback) when there is no GPU / library
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t = a.to(dtype=torch.float64)
        if not t.is_cuda:
            t = t.to(device or "cuda", non_blocking=True)
        return t.contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return torch.from_numpy(arr).to(device or "cuda")


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class BatchResult(NamedTuple):
    log_value: object
    value: object
    path: object


_ROUTES = {"hybrid": _lib.ROUTE_HYBRID, "series": _lib.ROUTE_SERIES,
           "integral": _lib.ROUTE_INTEGRAL}


def _launch_besselk(xd, nud, cfg: QuadratureConfig, route: int, want_value=True, want_path=True,
                    bins: int | None = None):
    torch = _torch()
    L = _lib.lib()
    n = xd.numel()
    logk = torch.empty_like(xd)
    k = torch.empty_like(xd) if want_value else None
    path = torch.empty(n, dtype=torch.uint8, device=xd.device) if want_path else None
    c = cfg.to_c(bins)
    with torch.cuda.device(xd.device):
        rc = L.bgk_besselk_batch(xd.data_ptr(), nud.data_ptr(), n, ctypes.byref(c), route,
                                 logk.data_ptr(), _ptr(k), _ptr(path), _stream_handle())
    _lib.check(rc, "bgk_besselk_batch")
    return logk, k, path


def bessel_k_batch(x, nu, cfg: QuadratureConfig = DEFAULT_CONFIG, route: str = "hybrid",
                   validate: bool = True) -> BatchResult:
    """K_nu(x) over arrays on the GPU.

    ``x`` and ``nu`` broadcast to a common shape.  CUDA tensors in give CUDA
    tensors out (no host round trip); anything else is copied to the device and
    the results come back as numpy arrays.  ``route``: "hybrid" (bessel_k),
    "series" (every element through the Temme path) or "integral" (the
    fixed-window quadrature with no threshold guard, like
    fixed_window_log_bessel_k).  With ``validate`` the EvalPoint / bessel_k
    domain rules are checked for the whole batch first (one device sync).
    """
    torch = _torch()
    if route not in _ROUTES:
        raise DomainError(f"route must be one of {sorted(_ROUTES)}")
    on_device = isinstance(x, torch.Tensor) and x.is_cuda
    if not on_device and not isinstance(nu, torch.Tensor):
        xa = np.asarray(x, dtype=np.float64)
        na = np.asarray(nu, dtype=np.float64)
        if xa.shape == na.shape and xa.size >= _HOST_PIPELINE_MIN:
            return _bessel_k_host_pipelined(xa, na, cfg, route, validate)
    xd = _to_device(x)
    nud = _to_device(nu, xd.device)
    if xd.shape != nud.shape:
        xd, nud = torch.broadcast_tensors(xd, nud)
        xd, nud = xd.contiguous(), nud.contiguous()
    shape = xd.shape
    xd, nud = xd.reshape(-1), nud.reshape(-1)
    if validate and xd.numel():
        _validate_batch(xd, nud, cfg, route)
    logk, k, path = _launch_besselk(xd, nud, cfg, _ROUTES[route])
    logk, k, path = logk.reshape(shape), k.reshape(shape), path.reshape(shape)
    if on_device:
        return BatchResult(logk, k, path)
    return BatchResult(logk.cpu().numpy(), k.cpu().numpy(), path.cpu().numpy())


def _bad_mask(xd, nud, cfg, route):
    torch = _torch()
    bad = ~torch.isfinite(xd) | (xd <= 0.0) | ~torch.isfinite(nud) | (nud < 0.0)
    if route == "series":
        bad |= xd >= cfg.small_x_threshold
    return bad


def _raise_for(xv: float, nv: float, cfg, route):
    EvalPoint(xv, nv)  # raises the reference's message for non-finite / negative
    if route == "series":
        raise DomainError(f"series path needs 0 < x < {cfg.small_x_threshold:g}, got {xv!r}")
    raise DomainError("x must be positive (r = 0 is handled by the Matern kernel)")


def _validate_batch(xd, nud, cfg, route):
    torch = _torch()
    bad = _bad_mask(xd, nud, cfg, route)
    if bool(bad.any()):
        i = int(torch.nonzero(bad)[0])
        _raise_for(float(xd[i]), float(nud[i]), cfg, route)


_HOST_CHUNK = 1 << 22  # elements per pipelined chunk for host (numpy) batches
_HOST_MIN_CHUNK = 1 << 20  # (A/B: 1M elements 1.25 ms as one chunk vs 1.7-2.5 ms as four; 4M 3.8-4.7 ms as four vs 4.4-5.0 ms as one)
# host batches from this size on take the pinned-staging path even as one chunk (1M
# elements on B200: 4.4 ms vs 6.0 ms through pageable copies; tools/bk_small_e2e.py)
_HOST_PIPELINE_MIN = 1 << 16


_STAGE: dict = {}  # per device: two pinned staging slots (x, nu) of _HOST_CHUNK elements
# per device: held for a whole pipelined call, so two host threads never stage into
# the same pinned slots (ctypes releases the GIL inside bgk_host_copy)
_STAGE_LOCKS: dict = {}
_STAGE_LOCKS_GUARD = threading.Lock()
_COPY_THREADS = None  # host threads of the pageable -> pinned staging copy (default: 3/4)


def _stage_slots(torch, dev):
    slots = _STAGE.get(dev.index)
    if slots is None:
        slots = [(torch.empty(_HOST_CHUNK, dtype=torch.float64, pin_memory=True),
                  torch.empty(_HOST_CHUNK, dtype=torch.float64, pin_memory=True))
                 for _ in range(2)]
        _STAGE[dev.index] = slots
    return slots


def _par_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src with host threads and non-temporal stores (bgk_host_copy):
    the staging copy is host-memory bound and paces the pipeline."""
    global _COPY_THREADS
    if _COPY_THREADS is None:
        import os

        try:
            ncpu = len(os.sched_getaffinity(0))
        except AttributeError:
            ncpu = os.cpu_count() or 1
        # 3/4 of the host threads: all of them oversubscribe the cores next to the
        # thread issuing the GPU work (64Mi batch on the 16-core box: 12 threads
        # 35-38 ms steadily, 16 threads 34-161 ms; tools/copy_threads.py)
        _COPY_THREADS = max(1, ncpu * 3 // 4)
    assert dst.dtype == src.dtype and dst.size == src.size and dst.flags.c_contiguous \
        and src.flags.c_contiguous
    _lib.check(_lib.load_library().bgk_host_copy(dst.ctypes.data, src.ctypes.data, src.nbytes,
                                                 _COPY_THREADS), "bgk_host_copy")


def _bessel_k_host_pipelined(xa, na, cfg, route, validate):
    """Host arrays in / host arrays out, chunked so that the host-side copy of chunk
    i+1 into a pinned staging slot, its H2D, the kernel on chunk i and the D2H of
    chunk i-1 overlap (copy-in stream, compute stream, copy-out stream); results
    land directly in page-locked output arrays."""
    torch = _torch()
    _lib.lib()
    shape = xa.shape
    xf = np.ascontiguousarray(xa).reshape(-1)
    nf = np.ascontiguousarray(na).reshape(-1)
    n = xf.size
    dev = torch.device("cuda", torch.cuda.current_device())
    with _STAGE_LOCKS_GUARD:
        lock = _STAGE_LOCKS.setdefault(dev.index, threading.Lock())
    with lock:
        return _host_pipeline_locked(torch, dev, xf, nf, n, shape, cfg, route, validate)


def _host_pipeline_locked(torch, dev, xf, nf, n, shape, cfg, route, validate):
    out_l = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out_k = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out_p = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    comp = torch.cuda.current_stream(dev)
    inp = torch.cuda.Stream(dev)
    copy = torch.cuda.Stream(dev)
    slots = _stage_slots(torch, dev)
    bad_any = None  # device flag: some element failed validation
    staged = [None, None]  # event: the slot's H2D has finished (slot reusable)
    freed = [None, None]   # event: the chunk's D2H has finished (device buffers reusable)
    # batches under four full chunks are cut into four, so their H2D, kernel and D2H
    # still overlap (at least _HOST_MIN_CHUNK elements per chunk)
    chunk = min(_HOST_CHUNK, max(_HOST_MIN_CHUNK, -(-n // 4)))
    for ci, c0 in enumerate(range(0, n, chunk)):
        c1 = min(n, c0 + chunk)
        s = ci % 2
        if staged[s] is not None:
            staged[s].synchronize()
        sx, sn = slots[s]
        _par_copy(sx.numpy()[:c1 - c0], xf[c0:c1])
        _par_copy(sn.numpy()[:c1 - c0], nf[c0:c1])
        with torch.cuda.stream(inp):
            if freed[s] is not None:
                inp.wait_event(freed[s])
            xd = sx[:c1 - c0].to(dev, non_blocking=True)
            nd = sn[:c1 - c0].to(dev, non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(inp)
        staged[s] = ev_in
        comp.wait_event(ev_in)
        xd.record_stream(comp)
        nd.record_stream(comp)
        if validate:  # deferred: one device flag for the whole call, no per-chunk sync
            b = _bad_mask(xd, nd, cfg, route).any()
            bad_any = b if bad_any is None else bad_any | b
        logk, k, path = _launch_besselk(xd, nd, cfg, _ROUTES[route])
        done = torch.cuda.Event()
        done.record(comp)
        copy.wait_event(done)
        with torch.cuda.stream(copy):
            out_l[c0:c1].copy_(logk, non_blocking=True)
            out_k[c0:c1].copy_(k, non_blocking=True)
            out_p[c0:c1].copy_(path, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        # keep the chunk's device buffers alive until its D2H has been issued/done
        logk.record_stream(copy)
        k.record_stream(copy)
        path.record_stream(copy)
        freed[s] = ev
    copy.synchronize()
    if bad_any is not None and bool(bad_any):
        # the first offending element, in order, gets the reference's message
        bad = ~np.isfinite(xf) | (xf <= 0.0) | ~np.isfinite(nf) | (nf < 0.0)
        if route == "series":
            bad |= xf >= cfg.small_x_threshold
        i = int(np.flatnonzero(bad)[0])
        _raise_for(float(xf[i]), float(nf[i]), cfg, route)
    return BatchResult(out_l.numpy().reshape(shape), out_k.numpy().reshape(shape),
                       out_p.numpy().reshape(shape))


_CFG_C: dict = {}  # (cfg, bins) -> bgk_config, built once


def _scalar_logk(x: float, nu: float, cfg: QuadratureConfig, route: int,
                 bins: int | None = None) -> float:
    """One evaluation on the current device: bgk_besselk_scalar (inputs and result
    through a mapped page-locked slot, one launch + one sync, no torch tensors)."""
    L = _lib.lib()
    key = (cfg, bins)
    c = _CFG_C.get(key)
    if c is None:
        c = _CFG_C.setdefault(key, cfg.to_c(bins))
    out = ctypes.c_double()
    _lib.check(L.bgk_besselk_scalar(float(x), float(nu), ctypes.byref(c), route,
                                    ctypes.byref(out), _stream_handle()), "bgk_besselk_scalar")
    return out.value


# ---------------------------------------------------------------------------------------
# public API (besselk.py:94-165)
# ---------------------------------------------------------------------------------------

def temme_pair(x: float, mu: float, cfg: QuadratureConfig = DEFAULT_CONFIG) -> tuple[float, float]:
    """Starting values (K_mu(x), K_{mu+1}(x)) for -0.5 <= mu < 0.5."""
    if not 0.0 < x < cfg.small_x_threshold:
        raise DomainError(f"temme_pair needs 0 < x < {cfg.small_x_threshold:g}, got {x!r}")
    if not -0.5 <= mu < 0.5:
        raise DomainError(f"mu must lie in [-0.5, 0.5), got {mu!r}")
    s0, s1, _ = temme_sums_batch([x], [mu], cfg)
    return float(s0[0]), (2.0 / x) * float(s1[0])


def temme_sums_batch(x, mu, cfg: QuadratureConfig = DEFAULT_CONFIG):
    """kernels.temme_sums over arrays: (s0, s1, terms), K_mu = s0, K_{mu+1} = (2/x) s1."""
    torch = _torch()
    L = _lib.lib()
    on_device = isinstance(x, torch.Tensor) and x.is_cuda
    xd = _to_device(x).reshape(-1)
    mud = _to_device(mu, xd.device).reshape(-1)
    s0 = torch.empty_like(xd)
    s1 = torch.empty_like(xd)
    terms = torch.empty(xd.numel(), dtype=torch.int64, device=xd.device)
    c = cfg.to_c()
    with torch.cuda.device(xd.device):
        rc = L.bgk_temme_sums_batch(xd.data_ptr(), mud.data_ptr(), xd.numel(), ctypes.byref(c),
                                    s0.data_ptr(), s1.data_ptr(), terms.data_ptr(),
                                    _stream_handle())
    _lib.check(rc, "bgk_temme_sums_batch")
    if on_device:
        return s0, s1, terms
    return s0.cpu().numpy(), s1.cpu().numpy(), terms.cpu().numpy()


def bessel_k_series(p: EvalPoint, cfg: QuadratureConfig = DEFAULT_CONFIG) -> BesselResult:
    """Series path: Temme sums plus forward recurrence, log-domain."""
    if not 0.0 < p.x < cfg.small_x_threshold:
        raise DomainError(
            f"series path needs 0 < x < {cfg.small_x_threshold:g}, got {p.x!r}")
    log_k = _scalar_logk(p.x, p.nu, cfg, _lib.ROUTE_SERIES)
    return _result(log_k, PathTaken.SERIES, p)


def _log_integrand_call(t: float, p: EvalPoint, order: int) -> float:
    torch = _torch()
    L = _lib.lib()
    td = _to_device([t])
    xd = _to_device([p.x], td.device)
    nd = _to_device([p.nu], td.device)
    out = torch.empty_like(td)
    with torch.cuda.device(td.device):
        rc = L.bgk_log_integrand_batch(td.data_ptr(), xd.data_ptr(), nd.data_ptr(), 1, order,
                                       out.data_ptr(), _stream_handle())
    _lib.check(rc, "bgk_log_integrand_batch")
    return float(out.cpu()[0])


def log_integrand(t: float, p: EvalPoint) -> float:
    """g(t) = log cosh(nu t) - x cosh(t)."""
    if t < 0.0:
        raise DomainError("t must be nonnegative")
    if p.x <= 0.0:
        raise DomainError("x must be positive")
    return _log_integrand_call(t, p, 0)


def log_integrand_d1(t: float, p: EvalPoint) -> float:
    if t < 0.0:
        raise DomainError("t must be nonnegative")
    return _log_integrand_call(t, p, 1)


def log_integrand_d2(t: float, p: EvalPoint) -> float:
    if t < 0.0:
        raise DomainError("t must be nonnegative")
    return _log_integrand_call(t, p, 2)


def fixed_window_log_bessel_k(x: float, nu: float,
                              cfg: QuadratureConfig = DEFAULT_CONFIG,
                              bins: int | None = None) -> float:
    """Raw fixed-window log K with no threshold guard.

    The bound audit and the pure-integral accuracy study deliberately apply
    this below the series threshold.
    """
    if x <= 0.0:
        raise DomainError("x must be positive")
    b = cfg.bins if bins is None else int(bins)
    return _scalar_logk(x, nu, cfg, _lib.ROUTE_INTEGRAL, bins=b)


def bessel_k_integral(p: EvalPoint, cfg: QuadratureConfig = DEFAULT_CONFIG) -> BesselResult:
    """Integral path over the fixed window [t_lower, t_upper]."""
    if p.x < cfg.small_x_threshold:
        raise DomainError(
            f"integral path needs x >= {cfg.small_x_threshold:g}, got {p.x!r}")
    log_k = fixed_window_log_bessel_k(p.x, p.nu, cfg)
    return _result(log_k, PathTaken.INTEGRAL, p)


def bessel_k(p: EvalPoint, cfg: QuadratureConfig = DEFAULT_CONFIG) -> BesselResult:
    """K_nu(x): series below the threshold, fixed-window quadrature at and
    above it (the boundary belongs to the integral side)."""
    if p.x <= 0.0:
        raise DomainError("x must be positive (r = 0 is handled by the Matern kernel)")
    if p.x < cfg.small_x_threshold:
        return bessel_k_series(p, cfg)
    return bessel_k_integral(p, cfg)
