"""Matern covariance engine -- the SPEC's covariance-engine API on the B200 kernels.

The reference package specifies this module but ships only its
compute kernel, ``kernels.matern_tile`` (kernels.py:338-381).  This module is
the caller, built around the sm_100a tile kernel of libbesselgp_sm100a.so:

  * ``MaternParams`` / ``LocationSet`` / ``TileSpec`` / ``CovarianceMatrix``
     with the SPEC's validation;
  * ``matern``, ``generate_tile`` (:315-323),
    ``generate_covariance`` (:324-332), ``normalize_locations`` (:288-296),
    ``morton_order`` (:297-305);
  * ``matern_tile`` with exactly the reference kernel's argument list.

Entry values are pure functions of the location pair and the parameters, so a
matrix is bitwise independent of tile size, layout, row sharding and launch
geometry, and symmetric bitwise.
"""

from __future__ import annotations

import ctypes
import enum
import math
import struct
import threading
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .besselk import DEFAULT_CONFIG, DomainError, QuadratureConfig

LN2 = 0.6931471805599453


# ---------------------------------------------------------------------------------------
# types
# ---------------------------------------------------------------------------------------

@dataclass(frozen=True)
class MaternParams:
    """(sigma^2, beta, nu): variance, range and smoothness; all finite and > 0."""

    sigma_sq: float
    beta: float
    nu: float

    def __post_init__(self):
        for name in ("sigma_sq", "beta", "nu"):
            v = getattr(self, name)
            if not (isinstance(v, (int, float, np.floating)) and math.isfinite(v) and v > 0.0):
                raise DomainError(f"{name} must be finite and positive, got {v!r}")


class Ordering(enum.Enum):
    AS_LOADED = "as_loaded"
    MORTON = "morton"


@dataclass(frozen=True, eq=False)
class LocationSet:
    """Ordered 2D coordinates (N x 2 float64)."""

    coords: np.ndarray
    normalized: bool = False
    ordering: Ordering = Ordering.AS_LOADED
    reject_duplicates: bool = field(default=True, compare=False)

    def __post_init__(self):
        c = np.ascontiguousarray(self.coords, dtype=np.float64)
        if c.ndim != 2 or c.shape[1] != 2:
            raise DomainError(f"coords must have shape (N, 2), got {c.shape}")
        if not np.all(np.isfinite(c)):
            raise DomainError("coords must be finite")
        if self.normalized and c.size and (c.min() < 0.0 or c.max() > 1.0):
            raise DomainError("normalized coords must lie in [0, 1]")
        if self.reject_duplicates and c.shape[0] > 1:
            u = np.unique(c, axis=0)
            if u.shape[0] != c.shape[0]:
                raise DomainError("duplicate locations are rejected at load (SPEC.md:276)")
        object.__setattr__(self, "coords", c)

    def __len__(self) -> int:
        return self.coords.shape[0]

    @property
    def x(self) -> np.ndarray:
        return np.ascontiguousarray(self.coords[:, 0])

    @property
    def y(self) -> np.ndarray:
        return np.ascontiguousarray(self.coords[:, 1])


@dataclass(frozen=True)
class TileSpec:
    row_offset: int
    col_offset: int
    rows: int
    cols: int
    tile_size: int = 256

    def __post_init__(self):
        if min(self.row_offset, self.col_offset, self.rows, self.cols) < 0:
            raise DomainError("TileSpec offsets and sizes must be nonnegative")
        if self.tile_size < 1:
            raise DomainError("tile_size must be at least 1")


@dataclass(eq=False)
class CovarianceMatrix:
    """Dense symmetric N x N matrix (or a row block / packed lower tiles of one).

    layout "full":  ``data`` is (row_end - row_begin) x N, row-major (numpy C
                    order or a CUDA tensor); rows [row_begin, row_end).
    layout "lower_tiles": ``data`` is (ntiles, ts, ts); tile l = p(p+1)/2 + q is
                    tile (p, q), q <= p, stored column-major within the tile
                    (SPEC.md:283), i.e. data[l].T is the tile.
    """

    N: int
    data: object
    layout: str = "full"
    tile_size: int = 256
    row_begin: int = 0
    row_end: int | None = None
    tile_begin: int = 0
    params: MaternParams | None = None

    def __post_init__(self):
        if self.row_end is None:
            self.row_end = self.N

    def to_numpy(self) -> np.ndarray:
        d = self.data
        if hasattr(d, "detach"):
            d = d.detach().cpu().numpy()
        return np.asarray(d)

    def tile(self, p: int, q: int) -> np.ndarray:
        """Tile (p, q) of the full matrix as an (m, n) array (any layout)."""
        ts, N = self.tile_size, self.N
        r0, c0 = p * ts, q * ts
        m, n = min(ts, N - r0), min(ts, N - c0)
        if not (0 <= r0 < N and 0 <= c0 < N):
            raise DomainError(f"tile ({p}, {q}) lies outside the {N} x {N} matrix")
        if self.layout == "full":
            if not (self.row_begin <= r0 and r0 + m <= self.row_end):
                raise DomainError(f"tile row {p} (rows [{r0}, {r0 + m})) is outside this "
                                  f"block's rows [{self.row_begin}, {self.row_end})")
            a = self.to_numpy()
            return a[r0 - self.row_begin:r0 - self.row_begin + m, c0:c0 + n]
        if q > p:
            return self.tile(q, p).T
        l = p * (p + 1) // 2 + q - self.tile_begin
        data = self.to_numpy()
        if not 0 <= l < data.shape[0]:
            raise DomainError(f"tile ({p}, {q}) is outside this shard's tile range "
                              f"[{self.tile_begin}, {self.tile_begin + data.shape[0]})")
        return data[l].T[:m, :n]

    # ---- CVMX binary format: 'CVMX', u32 version=1, u64 N, col-major f64 ----
    def write_cvmx(self, path: str) -> None:
        if self.layout != "full" or self.row_begin != 0 or self.row_end != self.N:
            raise DomainError("CVMX holds a complete full-layout matrix")
        a = self.to_numpy()
        with open(path, "wb") as fh:
            fh.write(b"CVMX" + struct.pack("<IQ", 1, self.N))
            # column-major == transpose of row-major; Sigma is symmetric bitwise
            np.ascontiguousarray(a.T).astype("<f8", copy=False).tofile(fh)

    # ---- CSV: row-major, 17 significant digits ------------------------
    def write_csv(self, path: str) -> None:
        if self.layout != "full":
            raise DomainError("CSV holds a full-layout matrix (or row block)")
        np.savetxt(path, self.to_numpy(), fmt="%.17g", delimiter=",")

    @staticmethod
    def read_csv(path: str) -> "CovarianceMatrix":
        a = np.atleast_2d(np.loadtxt(path, delimiter=",", dtype=np.float64))
        if a.shape[0] != a.shape[1]:
            raise DomainError("CSV matrix must be square")
        return CovarianceMatrix(N=a.shape[0], data=a)

    @staticmethod
    def read_cvmx(path: str) -> "CovarianceMatrix":
        with open(path, "rb") as fh:
            head = fh.read(16)
            if len(head) != 16 or head[:4] != b"CVMX":
                raise DomainError("not a CVMX file")
            version, N = struct.unpack("<IQ", head[4:])
            if version != 1:
                raise DomainError(f"unsupported CVMX version {version}")
            a = np.fromfile(fh, dtype="<f8", count=N * N).reshape(N, N).T
        return CovarianceMatrix(N=N, data=np.ascontiguousarray(a))


# ---------------------------------------------------------------------------------------
# plans
# ---------------------------------------------------------------------------------------

_plan_cache: "OrderedDict[tuple, _lib.BgkMaternPlan]" = OrderedDict()
_plan_lock = threading.Lock()


def matern_plan(theta: MaternParams, cfg: QuadratureConfig = DEFAULT_CONFIG) -> _lib.BgkMaternPlan:
    """The per-(theta, cfg) plan: node tables, log-prefactor, Temme constants, u LUT."""
    key = (float(theta.sigma_sq), float(theta.beta), float(theta.nu), cfg)
    with _plan_lock:
        plan = _plan_cache.get(key)
        if plan is not None:
            _plan_cache.move_to_end(key)
            return plan
    L = _lib.load_library()
    plan = _lib.BgkMaternPlan()
    c = cfg.to_c()
    _lib.check(L.bgk_matern_plan_init(ctypes.byref(plan), float(theta.sigma_sq),
                                      float(theta.beta), float(theta.nu), ctypes.byref(c)),
               "bgk_matern_plan_init")
    with _plan_lock:
        _plan_cache[key] = plan
        while len(_plan_cache) > 64:
            _plan_cache.popitem(last=False)
    return plan


def _torch():
    import torch

    return torch


def _stream():
    return _torch().cuda.current_stream().cuda_stream


def _dev(a, device=None):
    _lib.lib()  # BackendUnavailable (not a CPU fallback) when there is no GPU / library
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t = a.to(dtype=torch.float64)
        if not t.is_cuda:
            t = t.to(device or "cuda")
        return t.contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device or "cuda")


def _coords(locs, device=None):
    """(x, y) float64 CUDA tensors from a LocationSet, an (N,2) array or tensor, on
    ``device`` (default: a CUDA tensor's own device, else the current device)."""
    _lib.lib()  # BackendUnavailable (not a CPU fallback) when there is no GPU / library
    torch = _torch()
    if isinstance(locs, LocationSet):
        c = locs.coords
    else:
        c = locs
    if isinstance(c, torch.Tensor):
        c = c.to(dtype=torch.float64)
        if device is not None:
            c = c.to(device)
        elif not c.is_cuda:
            c = c.cuda()
        if c.ndim != 2 or c.shape[1] != 2:
            raise DomainError(f"coords must have shape (N, 2), got {tuple(c.shape)}")
        return c[:, 0].contiguous(), c[:, 1].contiguous()
    c = np.ascontiguousarray(c, dtype=np.float64)
    if c.ndim != 2 or c.shape[1] != 2:
        raise DomainError(f"coords must have shape (N, 2), got {c.shape}")
    t = torch.from_numpy(np.ascontiguousarray(c.T)).to(device if device is not None else "cuda")
    return t[0], t[1]


def _target_device(out, device, locs):
    """The device a covariance call runs on: a CUDA ``out``'s, else ``device``, else a
    CUDA location tensor's, else the current device."""
    _lib.lib()  # BackendUnavailable (not a CPU fallback) when there is no GPU / library
    torch = _torch()
    if isinstance(out, torch.Tensor) and out.is_cuda:
        if device is not None and torch.device(device) != out.device:
            raise DomainError(f"out is on {out.device} but device={device!r} was requested")
        return out.device
    if device is not None:
        d = torch.device(device)
        if d.type != "cuda":
            raise DomainError(f"device must be a CUDA device, got {device!r}")
        return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())
    c = locs.coords if isinstance(locs, LocationSet) else locs
    if isinstance(c, torch.Tensor) and c.is_cuda:
        return c.device
    return torch.device("cuda", torch.cuda.current_device())


def _check_device_out(buf, shape, dev):
    torch = _torch()
    if not (isinstance(buf, torch.Tensor) and buf.dtype == torch.float64 and buf.device == dev
            and tuple(buf.shape) == tuple(shape) and buf.is_contiguous()):
        got = (f"{tuple(buf.shape)} {buf.dtype} on {buf.device}, contiguous={buf.is_contiguous()}"
               if isinstance(buf, torch.Tensor) else type(buf).__name__)
        raise DomainError(f"out must be a contiguous {tuple(shape)} float64 tensor on {dev}; "
                          f"got {got}")


def _zero_tile_padding(buf, N, ts, l0, l1):
    """Zero the entries of packed lower tiles that lie beyond N (edge tiles of the
    last tile row and column); the kernel writes only the m x n valid part."""
    r = N % ts
    if r == 0 or l1 <= l0:
        return
    T = -(-N // ts)
    a, b = max(l0, T * (T - 1) // 2), min(l1, T * (T + 1) // 2)  # tile row p = T - 1
    if a < b:
        buf[a - l0:b - l0, :, r:] = 0.0   # column-major inside a tile: [l, col, row]
    last = T * (T + 1) // 2 - 1           # the corner tile (T-1, T-1)
    if l0 <= last < l1:
        buf[last - l0, r:, :] = 0.0


def _tile_launch(plan, rx, ry, cx, cy, out, ld, layout):
    L = _lib.lib()
    torch = _torch()
    with torch.cuda.device(out.device):
        rc = L.bgk_matern_tile(ctypes.byref(plan), rx.data_ptr(), ry.data_ptr(), rx.numel(),
                               cx.data_ptr(), cy.data_ptr(), cx.numel(), out.data_ptr(), ld,
                               layout, _stream())
    _lib.check(rc, "bgk_matern_tile")


# ---------------------------------------------------------------------------------------
# operations
# ---------------------------------------------------------------------------------------

def matern_tile(out, rx, ry, cx, cy, sigma_sq, beta, nu, log_prefactor, c_nodes, a_nodes, h,
                small_x_threshold, eps, series_cap):
    """Drop-in for kernels.matern_tile (kernels.py:339-340): fills ``out`` (len(rx) x
    len(cx), a CUDA float64 tensor, C-contiguous) from explicit node tables."""
    torch = _torch()
    L = _lib.lib()
    if not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float64
            and out.is_contiguous()):
        raise DomainError("out must be a contiguous float64 CUDA tensor")
    c = np.ascontiguousarray(c_nodes, dtype=np.float64)
    a = np.ascontiguousarray(a_nodes, dtype=np.float64)
    if c.shape != a.shape:
        raise DomainError("c_nodes and a_nodes must have the same length")
    plan = _lib.BgkMaternPlan()
    _lib.check(L.bgk_matern_plan_init_tables(
        ctypes.byref(plan), float(sigma_sq), float(beta), float(nu), float(log_prefactor),
        c.ctypes.data, a.ctypes.data, c.size, float(h), float(small_x_threshold), float(eps),
        int(series_cap)), "bgk_matern_plan_init_tables")
    rxd, ryd = _dev(rx, out.device), _dev(ry, out.device)
    cxd, cyd = _dev(cx, out.device), _dev(cy, out.device)
    if tuple(out.shape) != (rxd.numel(), cxd.numel()):
        raise DomainError("out must have shape (len(rx), len(cx))")
    _tile_launch(plan, rxd, ryd, cxd, cyd, out, cxd.numel(), _lib.LAYOUT_ROW_MAJOR)


def matern_batch(r, theta: MaternParams, cfg: QuadratureConfig = DEFAULT_CONFIG):
    """Matern covariance of distances ``r`` (any shape) on the GPU."""
    torch = _torch()
    on_device = isinstance(r, torch.Tensor) and r.is_cuda
    rd = _dev(r)
    shape = rd.shape
    rd = rd.reshape(-1)
    if rd.numel() and bool(((rd < 0) | ~torch.isfinite(rd)).any()):
        raise DomainError("r must be finite and nonnegative")
    zero = torch.zeros(1, dtype=torch.float64, device=rd.device)
    out = torch.empty((1, rd.numel()), dtype=torch.float64, device=rd.device)
    if rd.numel():
        # distance from (0, 0) to (r_j, 0) is sqrt(r_j^2) == r_j exactly (IEEE RN)
        _tile_launch(matern_plan(theta, cfg), zero, zero, rd, torch.zeros_like(rd), out,
                     rd.numel(), _lib.LAYOUT_ROW_MAJOR)
    out = out.reshape(shape)
    return out if on_device else out.cpu().numpy()


def matern(r: float, theta: MaternParams, cfg: QuadratureConfig = DEFAULT_CONFIG) -> float:
    """sigma^2 / (2^(nu-1) Gamma(nu)) u^nu K_nu(u), u = r / beta; r == 0 -> sigma^2."""
    if not (math.isfinite(r) and r >= 0.0):
        raise DomainError(f"r must be finite and nonnegative, got {r!r}")
    if r == 0.0:
        return float(theta.sigma_sq)
    return float(matern_batch(np.array([r]), theta, cfg)[0])


def generate_tile(spec: TileSpec, rows_locs, cols_locs, theta: MaternParams,
                  cfg: QuadratureConfig = DEFAULT_CONFIG, layout: str = "row"):
    """One covariance tile: entry (i, j) = matern(|rows_i - cols_j|).  Returns an
    (spec.rows, spec.cols) array -- numpy, or a CUDA tensor if the location inputs
    are CUDA tensors.  ``layout="col"`` stores it column-major (a Fortran-ordered
    numpy array / a transposed tensor view), as SPEC.md:283 keeps tiles."""
    torch = _torch()
    dev = _target_device(None, None, rows_locs)
    rx, ry = _coords(rows_locs, dev)
    cx, cy = _coords(cols_locs, dev)
    if rx.numel() != spec.rows or cx.numel() != spec.cols:
        raise DomainError("location slices are inconsistent with the TileSpec dims")
    on_device = any(isinstance(v, torch.Tensor) and v.is_cuda for v in (rows_locs, cols_locs))
    m, n = spec.rows, spec.cols
    if layout == "row":
        out = torch.empty((m, n), dtype=torch.float64, device=rx.device)
        if m and n:
            _tile_launch(matern_plan(theta, cfg), rx, ry, cx, cy, out, n, _lib.LAYOUT_ROW_MAJOR)
        return out if on_device else out.cpu().numpy()
    if layout == "col":
        buf = torch.empty((n, m), dtype=torch.float64, device=rx.device)
        if m and n:
            _tile_launch(matern_plan(theta, cfg), rx, ry, cx, cy, buf, m, _lib.LAYOUT_COL_MAJOR)
        return buf.T if on_device else np.asfortranarray(buf.cpu().numpy().T)
    raise DomainError("layout must be 'row' or 'col'")


def _cov_launch(plan, lx, ly, N, r0, r1, out, ld, layout):
    L = _lib.lib()
    torch = _torch()
    with torch.cuda.device(out.device):
        rc = L.bgk_matern_covariance(ctypes.byref(plan), lx.data_ptr(), ly.data_ptr(), N, r0, r1,
                                     out.data_ptr(), ld, layout, _stream())
    _lib.check(rc, "bgk_matern_covariance")


def _lower_launch(plan, lx, ly, N, ts, l0, l1, out):
    L = _lib.lib()
    torch = _torch()
    with torch.cuda.device(out.device):
        rc = L.bgk_matern_lower_tiles(ctypes.byref(plan), lx.data_ptr(), ly.data_ptr(), N, ts, l0,
                                      l1, out.data_ptr(), _stream())
    _lib.check(rc, "bgk_matern_lower_tiles")


def lower_tile_count(N: int, tile_size: int) -> int:
    T = -(-N // tile_size)
    return T * (T + 1) // 2


def empty_host_matrix(rows: int, cols: int) -> np.ndarray:
    """Page-locked host buffer for a covariance result (fast device->host copies)."""
    torch = _torch()
    return torch.empty((rows, cols), dtype=torch.float64, pin_memory=True).numpy()


def generate_covariance(locs, theta: MaternParams, cfg: QuadratureConfig = DEFAULT_CONFIG,
                        tile_size: int = 256, *, layout: str = "full", device=None, out=None,
                        rows: tuple[int, int] | None = None,
                        tiles: tuple[int, int] | None = None,
                        host_block_bytes: int = 1 << 30) -> CovarianceMatrix:
    """Matern covariance matrix of ``locs``.

    layout "full" (default): rows ``rows=(r0, r1)`` (default all) of the dense
      matrix, row-major.  Lower tiles are computed once and mirrored; values
      do not depend on ``tile_size``.
    layout "lower_tiles": the packed lower-triangle tiles (p, q), q <= p, of size
      tile_size, column-major inside each tile; ``tiles=(l0, l1)`` selects a
      contiguous range of tile indices (a shard).

    Result placement: ``out`` (a CUDA tensor or a host numpy array of the right
    shape) if given; else a CUDA tensor on ``device`` if given; else a host
    numpy array, computed on the GPU in row blocks that are copied back while
    the next block computes.
    """
    torch = _torch()
    if isinstance(locs, LocationSet):
        N = len(locs)
    else:
        N = int(locs.shape[0])
    if tile_size < 1:
        raise DomainError("tile_size must be at least 1")
    dev = _target_device(out, device, locs)
    lx, ly = _coords(locs, dev)
    plan = matern_plan(theta, cfg)

    if layout == "lower_tiles":
        ntiles = lower_tile_count(N, tile_size)
        l0, l1 = tiles if tiles is not None else (0, ntiles)
        if not (0 <= l0 <= l1 <= ntiles):
            raise DomainError(f"tiles must satisfy 0 <= l0 <= l1 <= {ntiles}, got {(l0, l1)}")
        shape = (l1 - l0, tile_size, tile_size)
        host = not (isinstance(out, torch.Tensor) and out.is_cuda) and (out is not None
                                                                         or device is None)
        if out is not None and not host:
            buf = out
            _check_device_out(buf, shape, dev)
        else:
            buf = torch.empty(shape, dtype=torch.float64, device=dev)
            if out is not None and (out.shape != shape or out.dtype != np.float64):
                raise DomainError(f"out must be a {shape} float64 array")
        # the padding of edge tiles (entries beyond N) is defined: zero
        _zero_tile_padding(buf, N, tile_size, l0, l1)
        if l1 > l0 and N:
            _lower_launch(plan, lx, ly, N, tile_size, l0, l1, buf)
        data = buf
        if host:
            if out is None:
                data = buf.cpu().numpy()
            else:
                np.copyto(out, buf.cpu().numpy())
                data = out
        return CovarianceMatrix(N=N, data=data, layout="lower_tiles", tile_size=tile_size,
                                tile_begin=l0, params=theta)
    if layout != "full":
        raise DomainError("layout must be 'full' or 'lower_tiles'")

    r0, r1 = rows if rows is not None else (0, N)
    if not (0 <= r0 <= r1 <= N):
        raise DomainError(f"rows must satisfy 0 <= r0 <= r1 <= N, got {(r0, r1)}")
    nrows = r1 - r0
    device_out = (out is not None and isinstance(out, torch.Tensor) and out.is_cuda) or (
        out is None and device is not None)
    if device_out:
        buf = out if out is not None else torch.empty((nrows, N), dtype=torch.float64,
                                                      device=dev)
        _check_device_out(buf, (nrows, N), dev)
        if nrows and N:
            _cov_launch(plan, lx, ly, N, r0, r1, buf, N, _lib.LAYOUT_ROW_MAJOR)
        return CovarianceMatrix(N=N, data=buf, tile_size=tile_size, row_begin=r0, row_end=r1,
                                params=theta)

    # host result: row blocks computed on the device, copied back while the next computes
    host = out if out is not None else np.empty((nrows, N), dtype=np.float64)
    if host.shape != (nrows, N) or host.dtype != np.float64 or not host.flags.c_contiguous:
        raise DomainError(f"out must be a C-contiguous ({nrows}, {N}) float64 array")
    if nrows == N and N >= _MIRROR_MIN_N and _is_pinned(host):
        _full_host_lower_mirrored(plan, lx, ly, N, host, host_block_bytes)
    elif nrows and N:
        block = max(64, min(nrows, (host_block_bytes // (8 * N)) // 64 * 64))
        host_t = torch.from_numpy(host)
        comp = torch.cuda.current_stream(lx.device)
        copy = torch.cuda.Stream(lx.device)
        bufs = [torch.empty((block, N), dtype=torch.float64, device=lx.device) for _ in range(2)]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        copied = [None, None]
        for bi, b0 in enumerate(range(r0, r1, block)):
            b1 = min(r1, b0 + block)
            s = bi % 2
            if copied[s] is not None:
                comp.wait_event(copied[s])
            _cov_launch(plan, lx, ly, N, b0, b1, bufs[s], N, _lib.LAYOUT_ROW_MAJOR)
            done[s].record(comp)
            copy.wait_event(done[s])
            with torch.cuda.stream(copy):
                host_t[b0 - r0:b1 - r0].copy_(bufs[s][:b1 - b0], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
                copied[s] = ev
        copy.synchronize()
    return CovarianceMatrix(N=N, data=host, tile_size=tile_size, row_begin=r0, row_end=r1,
                            params=theta)


_MIRROR_MIN_N = 4096
_MIRROR_POOL = None
_MIRROR_DIRECT = None  # override of _mirror_direct_blocks (tests / tuning)
_MIRROR_THREADS = None  # host threads of the mirror (default: 3/4)
_MIRROR_REVERSE = True  # row blocks bottom-up (A/B: 0.800-0.818 vs 0.813-0.832 s, profiles/r02_microbench.md)


def _is_pinned(a: np.ndarray) -> bool:
    """True when ``a`` is page-locked memory CUDA can copy into asynchronously."""
    torch = _torch()
    try:
        return bool(torch.from_numpy(a).is_pinned())
    except (RuntimeError, TypeError, ValueError):
        return False


def _host_threads() -> int:
    import os

    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def _mirror_direct_blocks(N: int, block: int) -> int:
    """Row blocks of the UPPER triangle next to the diagonal that each block sends
    over PCIe directly (the host mirrors the rest): trades PCIe time for the
    mirror's host-memory traffic.  Default 0: on the B200 boxes PCIe is the
    bound (M100, tools/e2e_diag.py: w = 0 / 4 / 8 / 14 -> 0.874 / 0.876 / 0.932 /
    1.014 s; full rows 1.40 s)."""
    if _MIRROR_DIRECT is not None:
        return _MIRROR_DIRECT
    return 0


def host_d2h_bytes(N: int, rows=None, pinned: bool = True, host_block_bytes: int = 1 << 30) -> int:
    """Device-to-host bytes generate_covariance moves for a host-array result."""
    r0, r1 = rows if rows is not None else (0, N)
    if not (r0 == 0 and r1 == N and N >= _MIRROR_MIN_N and pinned):
        return 8 * (r1 - r0) * N
    block = max(64, min(N, (host_block_bytes // (8 * N)) // 64 * 64))
    w = _mirror_direct_blocks(N, block)
    return sum(8 * (min(N, b0 + block) - b0) * min(N, b0 + block + w * block)
               for b0 in range(0, N, block))


def _full_host_lower_mirrored(plan, lx, ly, N, host, block_bytes):
    """The whole N x N matrix into a page-locked host array with about half the
    PCIe traffic: per row block [b0, b1) the device computes the lower part plus w
    blocks of the upper one, cols [0, b1 + w block) (bitwise the entries of the
    full rows), a 2D copy moves just that part, and host threads mirror
    rows [b0, b1) x cols [0, b0 - w block) into rows [0, b0 - w block) x
    cols [b0, b1) while the next block computes and copies (the rows in between
    received those columns directly).  The mirror of block k writes only rows
    < b0, which no later copy touches."""
    global _MIRROR_POOL
    torch = _torch()
    L = _lib.lib()
    if _MIRROR_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _MIRROR_POOL = ThreadPoolExecutor(max_workers=1)  # mirrors in block order
    # 3/4 of the host threads: the mirror then keeps pace with the copies and leaves
    # DRAM bandwidth to the DMA (M100 on a 16-core box, tools/e2e_sweep.py, median of
    # 3 with 1 GiB blocks: 8 -> 0.890 s, 12 -> 0.820 s, 16 -> 0.894 s; round 1: 4 -> 1.4 s)
    nthreads = _MIRROR_THREADS or max(1, _host_threads() * 3 // 4)
    block = max(64, min(N, (block_bytes // (8 * N)) // 64 * 64))
    w = _mirror_direct_blocks(N, block)
    dev = lx.device
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    bufs = [torch.empty((block, N), dtype=torch.float64, device=dev) for _ in range(2)]
    copied = [None, None]
    futs = []
    hp = host.ctypes.data

    def mirror(ev, b0, b1):
        # rows [b0 - w block, b0) already hold cols [b0, b1): their blocks sent them
        ev.synchronize()
        _lib.check(L.bgk_host_mirror_block(hp, N, b0, b1, 0, max(0, b0 - w * block), nthreads),
                   "bgk_host_mirror_block")

    # largest blocks first (the mirror of the last block is the one left uncovered at
    # the end: make it the smallest).  Safe in either order: block k's copy writes
    # rows [b0, b1) x cols [0, b1), its mirror rows [0, b0) x cols [b0, b1) -- no
    # block's copy touches another block's mirror columns.
    order = list(range(0, N, block))
    if _MIRROR_REVERSE and w == 0:
        order.reverse()
    try:
        for bi, b0 in enumerate(order):
            b1 = min(N, b0 + block)
            s = bi % 2
            if copied[s] is not None:
                comp.wait_event(copied[s])
            ce = min(N, b1 + w * block)  # the lower part + w blocks of the upper
            _tile_launch(plan, lx[b0:b1], ly[b0:b1], lx[:ce], ly[:ce], bufs[s], N,
                         _lib.LAYOUT_ROW_MAJOR)
            done = torch.cuda.Event()
            done.record(comp)
            copy.wait_event(done)
            _lib.check(L.bgk_memcpy2d_d2h(hp + 8 * b0 * N, 8 * N, bufs[s].data_ptr(), 8 * N,
                                          8 * ce, b1 - b0, copy.cuda_stream), "bgk_memcpy2d_d2h")
            ev = torch.cuda.Event()
            ev.record(copy)
            copied[s] = ev
            futs.append(_MIRROR_POOL.submit(mirror, ev, b0, b1))
        copy.synchronize()
    finally:
        for f in futs:
            f.result()


# ---------------------------------------------------------------------------------------
# location preprocessing
# ---------------------------------------------------------------------------------------

def _is_cuda(a) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, torch.Tensor) and a.is_cuda


def normalize_locations_device(coords):
    """normalize_locations on the GPU for an (N, 2) CUDA tensor (bitwise equal to
    the host version); returns a new (N, 2) float64 CUDA tensor."""
    torch = _torch()
    L = _lib.lib()
    c = coords.to(dtype=torch.float64)
    x, y = c[:, 0].contiguous(), c[:, 1].contiguous()
    n = x.numel()
    if n == 0:
        raise DomainError("location set must be non-empty")
    bounds = torch.empty(4, dtype=torch.int64, device=x.device)
    ox, oy = torch.empty_like(x), torch.empty_like(y)
    with torch.cuda.device(x.device):
        _lib.check(L.bgk_normalize_locations(x.data_ptr(), y.data_ptr(), n, bounds.data_ptr(),
                                             ox.data_ptr(), oy.data_ptr(), _stream()),
                   "bgk_normalize_locations")
    b = bounds.cpu().numpy().view(np.uint64)  # order-mapped doubles -> doubles
    neg = (b >> np.uint64(63)) == 0
    raw_bits = np.where(neg, ~b, b & np.uint64(0x7FFFFFFFFFFFFFFF))
    mnx, mny, mxx, mxy = raw_bits.view(np.float64)
    if max(mxx - mnx, mxy - mny) == 0.0:
        raise DomainError("degenerate location set: all points coincide")
    return torch.stack([ox, oy], 1)


def morton_order_device(coords, bits_per_axis: int = 16):
    """(reordered coords, permutation) on the GPU for normalized (N, 2) CUDA coords:
    device Morton keys + a stable sort (ties keep the original order)."""
    torch = _torch()
    L = _lib.lib()
    if not 1 <= bits_per_axis <= 31:
        raise DomainError("bits_per_axis must lie in [1, 31]")
    c = coords.to(dtype=torch.float64)
    x, y = c[:, 0].contiguous(), c[:, 1].contiguous()
    keys = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        _lib.check(L.bgk_morton_keys(x.data_ptr(), y.data_ptr(), x.numel(), bits_per_axis,
                                     keys.data_ptr(), _stream()), "bgk_morton_keys")
    # keys use at most 62 bits, so signed int64 order == unsigned order
    perm = torch.sort(keys, stable=True).indices
    return c[perm], perm


def normalize_locations(raw):
    """Map into the unit square with one scale factor l = max(extent_x, extent_y).

    A LocationSet is normalized on the host; an (N, 2) CUDA tensor on the device
    (``normalize_locations_device``, bitwise equal)."""
    if _is_cuda(raw):
        return normalize_locations_device(raw)
    c = raw.coords
    if c.shape[0] == 0:
        raise DomainError("location set must be non-empty")
    mn = c.min(axis=0)
    ext = c.max(axis=0) - mn
    ell = float(max(ext[0], ext[1]))
    if ell == 0.0:
        raise DomainError("degenerate location set: all points coincide")
    out = (c - mn) / ell
    return LocationSet(np.clip(out, 0.0, 1.0), normalized=True, ordering=raw.ordering,
                       reject_duplicates=raw.reject_duplicates)


def _part1by1(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)
    return v


def morton_order(s, bits_per_axis: int = 16):
    """Z-order permutation: quantise to floor(c (2^bits - 1)), interleave with x in
    the low bit, stable sort (ties keep the original order).  Returns the
    reordered set and the permutation ``perm`` with new[i] = old[perm[i]].
    An (N, 2) CUDA tensor of normalized coordinates is ordered on the device."""
    if _is_cuda(s):
        return morton_order_device(s, bits_per_axis)
    if not s.normalized:
        raise DomainError("morton_order needs a normalized LocationSet")
    if not 1 <= bits_per_axis <= 31:
        raise DomainError("bits_per_axis must lie in [1, 31]")
    scale = float((1 << bits_per_axis) - 1)
    q = np.floor(s.coords * scale).astype(np.uint64)
    key = _part1by1(q[:, 0]) | (_part1by1(q[:, 1]) << np.uint64(1))
    perm = np.argsort(key, kind="stable")
    return (LocationSet(s.coords[perm], normalized=True, ordering=Ordering.MORTON,
                        reject_duplicates=False), perm)
