"""Where a scalar bessel_k(EvalPoint) call spends its time (GPU box): the raw C-ABI
call on the legacy default stream, the same with torch's current stream looked up per
call, and the public API.  usage: python tools/scalar_latency.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import _lib, besselk  # noqa: E402

L = _lib.lib()
c = besselk.DEFAULT_CONFIG.to_c()
out = ctypes.c_double()
N = 4000


def bench(fn):
    for _ in range(200):
        fn()
    t = time.perf_counter()
    for _ in range(N):
        fn()
    return (time.perf_counter() - t) / N * 1e6


for x, nu in [(0.05, 1.5), (2.0, 1.5), (30.0, 10.0)]:
    raw = bench(lambda: L.bgk_besselk_scalar(x, nu, ctypes.byref(c), 0, ctypes.byref(out), None))
    strm = bench(lambda: L.bgk_besselk_scalar(x, nu, ctypes.byref(c), 0, ctypes.byref(out),
                                              torch.cuda.current_stream().cuda_stream))
    p = bg.EvalPoint(x, nu)
    api = bench(lambda: bg.bessel_k(p))
    cs = bench(lambda: torch.cuda.current_stream().cuda_stream)
    print(f"x={x} nu={nu}: raw C call {raw:.2f} us, + current_stream {strm:.2f} us, "
          f"bessel_k {api:.2f} us (current_stream alone {cs:.2f} us)")
