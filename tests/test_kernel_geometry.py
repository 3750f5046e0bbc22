"""The Matern kernel's launch geometry on the B200: the design
assumes 4 resident 256-thread CTAs per SM (32 warps) for the plans the bench
runs -- the shared-memory budget (replicated exp table, tile, permutation,
histogram) is sized for it, and one byte too many silently drops to 3."""

import ctypes

import pytest

from paper_2502_00356_b200 import _lib


def _plan(nu):
    L = _lib.load_library()
    cfg = _lib.BgkConfig(0.0, 9.0, 40, 0.1, 15000, 2.0 ** -52)
    plan = _lib.BgkMaternPlan()
    assert L.bgk_matern_plan_init(ctypes.byref(plan), 1.0, 0.1, nu, ctypes.byref(cfg)) == 0
    return L, plan


@pytest.mark.gpu
@pytest.mark.parametrize("nu", [1.5, 0.5, 0.3, 0.8, 1.7, 2.9])
def test_matern_four_ctas_per_sm(nu):
    import torch

    torch.cuda.init()
    L, plan = _plan(nu)
    ctas, smem, regs = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = L.bgk_matern_kernel_info(ctypes.byref(plan), ctypes.byref(ctas), ctypes.byref(smem),
                                  ctypes.byref(regs))
    assert rc == 0, L.bgk_last_error()
    assert regs.value <= 64
    assert ctas.value == 4, f"nu={nu}: {ctas.value} CTAs/SM with {smem.value} B smem per CTA"
