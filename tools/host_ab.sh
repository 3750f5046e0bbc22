#!/bin/bash
# A/B of library variants on the host-buffer paths: BK 64Mi host arrays (5 calls) and
# the M100 host matrix (3 calls).  usage: bash tools/host_ab.sh ab/A.so ab/B.so
LIB=paper_2502_00356_b200/libbesselgp_sm100a.so
cp $LIB /tmp/lib_orig.so
for V in "$@" "$@"; do
  cp "$V" $LIB
  echo "== $V"
  python tools/bk_e2e_rep.py 2>&1 | head -2
  python - <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2502_00356_b200 as bg
N = 100_000
locs = np.random.default_rng(1).random((N, 2))
host = bg.empty_host_matrix(N, N)
ts = []
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    bg.generate_covariance(locs, bg.MaternParams(1.0, 0.1, 1.5), out=host)
    torch.cuda.synchronize(); ts.append(round(time.perf_counter() - t0, 3))
print("m100 host", ts)
PY
done
cp /tmp/lib_orig.so $LIB
