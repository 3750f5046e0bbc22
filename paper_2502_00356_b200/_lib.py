"""ctypes binding of libbesselgp_sm100a.so (declared in include/besselgp_b200.h).

The library is the ONLY compute backend: there is no CPU fallback.  If the
shared object is missing, or no CUDA device is visible, every entry point
raises ``BackendUnavailable`` instead of silently computing elsewhere.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libbesselgp_sm100a.so"
LIB_PATH = os.path.join(_HERE, LIB_NAME)

BGK_OK = 0
BGK_ABI_VERSION = 4
ROUTE_HYBRID, ROUTE_SERIES, ROUTE_INTEGRAL = 0, 1, 2
PATH_SERIES, PATH_INTEGRAL = 0, 1
LAYOUT_ROW_MAJOR, LAYOUT_COL_MAJOR = 0, 1
MAX_NODES = 1024
MAX_BUCKETS = 1024
MACRO_TILE = 64
MAX_PEERS = 32
IPC_HANDLE_BYTES = 64


class BackendUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is missing (no CPU fallback exists)."""


class BackendError(RuntimeError):
    """A library call returned a negative BGK_ERR_* status."""


class BgkConfig(ctypes.Structure):
    """bgk_config (mirrors QuadratureConfig, besselk.py:32-41)."""

    _fields_ = [
        ("t_lower", ctypes.c_double),
        ("t_upper", ctypes.c_double),
        ("bins", ctypes.c_int64),
        ("small_x_threshold", ctypes.c_double),
        ("series_cap", ctypes.c_int64),
        ("eps_machine", ctypes.c_double),
    ]


class BgkMaternPlan(ctypes.Structure):
    """bgk_matern_plan -- caller-allocated POD filled by bgk_matern_plan_init*."""

    _fields_ = [
        ("abi", ctypes.c_int32),
        ("nnodes", ctypes.c_int32),
        ("nbuckets", ctypes.c_int32),
        ("key_base", ctypes.c_int32),
        ("fast", ctypes.c_int32),
        ("m_steps", ctypes.c_int32),
        ("anchor_min", ctypes.c_int32),
        ("anchor_max", ctypes.c_int32),
        ("key_shift", ctypes.c_int32),
        ("nosub_buckets", ctypes.c_int32),
        ("pow_mode", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("pow_pref", ctypes.c_double),
        ("sigma_sq", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("nu", ctypes.c_double),
        ("log_prefactor", ctypes.c_double),
        ("h", ctypes.c_double),
        ("small_x_threshold", ctypes.c_double),
        ("eps_machine", ctypes.c_double),
        ("series_cap", ctypes.c_int64),
        ("mu", ctypes.c_double),
        ("gam1", ctypes.c_double),
        ("gam2", ctypes.c_double),
        ("fact", ctypes.c_double),
        ("gamma_1p_mu", ctypes.c_double),
        ("gamma_1m_mu", ctypes.c_double),
        ("c", ctypes.c_double * MAX_NODES),
        ("a", ctypes.c_double * MAX_NODES),
        ("aw", ctypes.c_double * MAX_NODES),
        ("lut", ctypes.c_uint32 * MAX_BUCKETS),
    ]


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
_int = ctypes.c_int

# symbol -> (restype, argtypes); kept in sync with include/besselgp_b200.h
SIGNATURES = {
    "bgk_besselk_batch": (_int, [_vp, _vp, _i64, ctypes.POINTER(BgkConfig), _int, _vp, _vp, _vp, _vp]),
    "bgk_besselk_scalar": (_int, [_d, _d, ctypes.POINTER(BgkConfig), _int,
                                  ctypes.POINTER(ctypes.c_double), _vp]),
    "bgk_besselk_windows_host": (_int, [_vp, _vp, _i64, ctypes.POINTER(BgkConfig), _vp, _vp, _vp]),
    "bgk_besselk_windows": (_int, [_vp, _vp, _i64, ctypes.POINTER(BgkConfig), _vp, _vp, _vp, _vp]),
    "bgk_temme_sums_batch": (_int, [_vp, _vp, _i64, ctypes.POINTER(BgkConfig), _vp, _vp, _vp, _vp]),
    "bgk_log_integrand_batch": (_int, [_vp, _vp, _vp, _i64, _int, _vp, _vp]),
    "bgk_matern_plan_size": (ctypes.c_size_t, []),
    "bgk_matern_plan_init": (_int, [ctypes.POINTER(BgkMaternPlan), _d, _d, _d, ctypes.POINTER(BgkConfig)]),
    "bgk_matern_plan_init_tables": (_int, [ctypes.POINTER(BgkMaternPlan), _d, _d, _d, _d, _vp, _vp,
                                           _i64, _d, _d, _d, _i64]),
    "bgk_matern_tile": (_int, [ctypes.POINTER(BgkMaternPlan), _vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64,
                               _int, _vp]),
    "bgk_matern_covariance": (_int, [ctypes.POINTER(BgkMaternPlan), _vp, _vp, _i64, _i64, _i64, _vp, _i64,
                                     _int, _vp]),
    "bgk_matern_lower_tiles": (_int, [ctypes.POINTER(BgkMaternPlan), _vp, _vp, _i64, _i64, _i64, _i64,
                                      _vp, _vp]),
    "bgk_last_error": (ctypes.c_char_p, []),
    "bgk_abi_version": (_int, []),
    "bgk_launch_count": (_i64, []),
    "bgk_debug_set_device_alias": (_int, [_int]),
    "bgk_fp64_probe": (_int, [_vp, _i64, _int, _vp, ctypes.POINTER(ctypes.c_double)]),
    "bgk_sqrt_rn_check": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "bgk_matern_phase_profile": (_int, [_vp, _int]),
    "bgk_matern_kernel_info": (_int, [ctypes.POINTER(BgkMaternPlan), ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "bgk_matern_covariance_peer": (_int, [ctypes.POINTER(BgkMaternPlan), _vp, _vp, _i64, _int,
                                          ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_void_p), _i64, _i64, _vp]),
    "bgk_matern_covariance_peer_band": (_int, [ctypes.POINTER(BgkMaternPlan), _vp, _vp, _i64, _int,
                                               ctypes.POINTER(ctypes.c_int64),
                                               ctypes.POINTER(ctypes.c_void_p), _int, _vp]),
    "bgk_memcpy2d_d2h": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp]),
    "bgk_host_mirror_lower": (_int, [_vp, _i64, _i64, _i64, _int]),
    "bgk_host_copy": (_int, [_vp, _vp, _i64, _int]),
    "bgk_host_mirror_block": (_int, [_vp, _i64, _i64, _i64, _i64, _i64, _int]),
    "bgk_ipc_export": (_int, [_vp, _vp, ctypes.POINTER(ctypes.c_uint64)]),
    "bgk_ipc_open": (_int, [_vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "bgk_ipc_close": (_int, [_vp, ctypes.c_uint64]),
    "bgk_enable_peer_access": (_int, [_int]),
    "bgk_can_access_peer": (_int, [_int, ctypes.POINTER(ctypes.c_int)]),
    "bgk_normalize_locations": (_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "bgk_morton_keys": (_int, [_vp, _vp, _i64, _int, _vp, _vp]),
    "bgk_log_grid": (_int, [_vp, _i64, _vp, _i64, ctypes.POINTER(BgkConfig), _int, _i64, _int, _vp,
                            _vp]),
}

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the sm_100a library in place with nvcc (cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", _HERE] + (["-B"] if force else []), check=True)
    return LIB_PATH


# test / profiling hooks, not compute entry points: tolerated missing so that
# tools/ab_libs.sh can time libraries built from older revisions
_INTROSPECTION = {"bgk_matern_kernel_info", "bgk_matern_phase_profile"}


def load_library():
    """Load the shared object and bind every exported symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendUnavailable(
                    f"{LIB_NAME} is not built; run `make -C {_HERE}` or __graft_entry__.build() "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                if name in _INTROSPECTION and not hasattr(lib, name):
                    continue  # profiling hooks only (an older library in an A/B run)
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.bgk_abi_version() != BGK_ABI_VERSION:
                raise BackendUnavailable("ABI version mismatch between library and bindings")
            if lib.bgk_matern_plan_size() != ctypes.sizeof(BgkMaternPlan):
                raise BackendUnavailable("bgk_matern_plan layout mismatch")
            _lib = lib
    return _lib


_cuda_ok = False


def lib():
    """The bound library, after checking a CUDA device is present."""
    global _cuda_ok
    if _cuda_ok:
        return _lib
    import torch

    L = load_library()
    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device visible: the sm_100a kernels are the only backend")
    _cuda_ok = True
    return L


def check(rc: int, what: str) -> None:
    if rc != BGK_OK:
        msg = load_library().bgk_last_error().decode(errors="replace")
        raise BackendError(f"{what} failed (status {rc}): {msg}")


def launch_count() -> int:
    return int(load_library().bgk_launch_count())
