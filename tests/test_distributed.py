"""Multi-process (world_size 2, gloo, CPU) tests of the sharding plumbing in
paper_2502_00356_b200/distributed.py.  The CPU oracle stands in for the GPU
compute (it is the checker here, injected through ``compute=``); what is under
test is the shard arithmetic, the row-block assembly and the gathers."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ORACLE_DIR, ROOT

from paper_2502_00356_b200 import distributed as D


def test_shard_arithmetic():
    for N in (1, 7, 1000, 100_000):
        for G in (1, 2, 3, 4, 8):
            sh = D.row_shards(N, G)
            assert sh[0][0] == 0 and sh[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            assert max(r1 - r0 for r0, r1 in sh) - min(r1 - r0 for r0, r1 in sh) <= 1
            tot = sum(D.computed_entries(N, r0, r1) for r0, r1 in sh)
            # diagonal blocks once per pair, everything else once per entry
            assert tot == N * N - sum((r1 - r0) * (r1 - r0 - 1) // 2 for r0, r1 in sh)
    # packed lower tiles of the N=200K layout: equal-count contiguous shards
    T = -(-200_000 // 256)
    nt = T * (T + 1) // 2
    assert nt == 306_153
    sh = [D.tile_shard(nt, 8, g) for g in range(8)]
    assert sh[0][0] == 0 and sh[-1][1] == nt and max(b - a for a, b in sh) - min(b - a for a, b in sh) <= 1
    with pytest.raises(ValueError):
        D.row_shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, ORACLE_DIR)
    import oracle  # checker / CPU stand-in for the kernel

    from paper_2502_00356_b200 import distributed as Dd

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)
        N = 203
        locs = rng.random((N, 2))

        def compute(lc, theta, cfg, rows):
            return torch.from_numpy(oracle.generate_covariance(lc, 1.0, 0.1, 1.5, row_range=rows))

        r0, r1, blk = Dd.generate_covariance_sharded(locs, None, compute=compute)
        assert (r0, r1) == Dd.row_shard(N, world, rank)
        full = Dd.gather_rows(blk, N, dst=0)
        ok = True
        if rank == 0:
            ref = oracle.generate_covariance(locs, 1.0, 0.1, 1.5)
            ok = bool(np.array_equal(full.numpy(), ref))
        else:
            ok = full is None

        x = 140.0 * (1.0 - rng.random(1001))
        nu = 20.0 * (1.0 - rng.random(1001))

        def bk(xs, ns, cfg):
            return torch.from_numpy(oracle.refined_log_bessel_batch(xs, ns))

        i0, i1, lk = Dd.bessel_k_batch_sharded(x, nu, gather=True, compute=bk)
        ok = ok and (i0, i1) == (0, 1001)
        ok = ok and bool(np.array_equal(lk.numpy(), oracle.refined_log_bessel_batch(x, nu)))
        with open(os.path.join(result_dir, f"r{rank}"), "w") as fh:
            fh.write("ok" if ok else "bad")
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_and_gathers(tmp_path, oracle):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    for r in range(world):
        assert open(os.path.join(tmp_path, f"r{r}")).read() == "ok"
