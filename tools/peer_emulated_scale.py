"""Emulated multi-GPU run of the fused peer-band kernel at M100 scale on ONE GPU.

G owner row blocks live on this device and every rank's share (its cyclic half band
of 64x64 tile pairs, direct stores into its own block, mirrors into the other
owners' blocks) is launched and timed on its own (CUDA events).  With one GPU per
rank the ranks run concurrently, so max_g t_g is the compute time an G-GPU run would
see before NVLink effects (here the "remote" mirror stores land in local HBM).  The
union of the blocks is checked against the single-GPU matrix on sampled rows.
Not a scaling measurement -- an emulation of the per-rank work split.

usage: python tools/peer_emulated_scale.py [N] [G ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_00356_b200 as bg  # noqa: E402
from paper_2502_00356_b200 import distributed as D  # noqa: E402
from paper_2502_00356_b200.besselk import DEFAULT_CONFIG  # noqa: E402
from paper_2502_00356_b200.covariance import _coords, matern_plan  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
Gs = [int(g) for g in sys.argv[2:]] or [1, 2, 4, 8]
locs = np.random.default_rng(20250201).random((N, 2))
theta = bg.MaternParams(1.0, 0.1, 1.5)
lx, ly = _coords(locs)
plan = matern_plan(theta, DEFAULT_CONFIG)
rng = np.random.default_rng(3)
rows = np.unique(np.concatenate([[0, 63, 64, N - 1], rng.integers(0, N, 12)]))

full = bg.generate_covariance(locs, theta, device="cuda").data
ref_rows = full[torch.from_numpy(rows).cuda()].clone()
del full
torch.cuda.empty_cache()
res = []
for G in Gs:
    starts = D.macro_row_starts(N, G)
    blocks = []
    for g in range(G):
        r0, r1 = D.owner_rows(N, G, g)
        blocks.append(torch.empty((r1 - r0, N), dtype=torch.float64, device="cuda"))
    bases = [b.data_ptr() if b.numel() else 1 for b in blocks]
    for g in range(G):  # warm-up
        D._launch_peer(plan, lx, ly, N, starts, bases, 0, 0, rank=g)
    torch.cuda.synchronize()
    times = []
    for g in range(G):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            D._launch_peer(plan, lx, ly, N, starts, bases, 0, 0, rank=g)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 2)
    got = []
    for r in rows:
        g = max(i for i in range(G) if D.owner_rows(N, G, i)[0] <= r)
        got.append(blocks[g][r - D.owner_rows(N, G, g)[0]])
    ok = bool(torch.equal(torch.stack(got), ref_rows))
    mirror = [D.peer_mirror_bytes(N, G, g) for g in range(G)] if hasattr(D, "peer_mirror_bytes") else None
    res.append({"G": G, "rank_kernel_ms": [round(t, 3) for t in times], "max_ms": round(max(times), 3),
                "sum_ms": round(sum(times), 3), "union_equals_single_gpu_rows": ok,
                "mirror_bytes_per_rank": mirror})
    print(json.dumps(res[-1]), flush=True)
    del blocks
    torch.cuda.empty_cache()
t1 = res[0]["max_ms"] if res and res[0]["G"] == 1 else None
for r in res:
    if t1:
        r["emulated_speedup_vs_G1"] = round(t1 / r["max_ms"], 3)
print(json.dumps({"N": N, "emulation": "per-rank kernels on one GPU, remote stores local", "runs": res}))
