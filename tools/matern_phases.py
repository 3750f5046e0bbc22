"""Where the Matern kernel's warps spend their cycles, per task-loop phase.

Needs a library built with -DBGK_MATERN_PROFILE=1 (bash tools/build_variant.sh P WT
-DBGK_MATERN_PROFILE=1), swapped in as the package library.  Runs one N x N
covariance (default N = 40000, nu = 1.5; a full-matrix launch like M100) and prints,
for each of the six barriers of the task loop, the share of warp-cycles spent working
before it and waiting at it.
usage: python tools/matern_phases.py [N] [nu]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import _lib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
nu = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5
L = _lib.lib()
out = (ctypes.c_double * 12)()
locs = np.random.default_rng(20250201).random((N, 2))
theta = bg.MaternParams(1.0, 0.1, nu)
bg.generate_covariance(locs, theta, device="cuda:0")  # warm-up
torch.cuda.synchronize()
assert L.bgk_matern_phase_profile(out, 1) == 0, L.bgk_last_error()
bg.generate_covariance(locs, theta, device="cuda:0")
torch.cuda.synchronize()
assert L.bgk_matern_phase_profile(out, 1) == 0
v = np.array(out[:])
tot = v.sum()
names = ["classify", "scan (1st half)", "scan (2nd half)", "scatter", "compute", "store + prep"]
print(f"N={N} nu={nu}: warp-cycles {tot:.4g}")
for i, nm in enumerate(names):
    print(f"  {nm:18s} work {100 * v[2 * i] / tot:5.1f}%   wait at barrier {100 * v[2 * i + 1] / tot:5.1f}%")
print(f"  total wait {100 * v[1::2].sum() / tot:5.1f}%")
