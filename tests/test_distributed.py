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


@pytest.mark.parametrize("T", [1, 2, 3, 4, 7, 8, 31, 64])
@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_peer_band_covers_every_tile_pair_once(T, G):
    """The cyclic half band (bgk_matern_covariance_peer_band): over all ranks every
    unordered macro-tile pair {p, q} is computed exactly once, each rank's direct
    stores stay in its own rows, and the work is balanced."""
    N = 64 * T
    s = D.macro_row_starts(N, G)
    seen = {}
    for h in range(G):
        for p in range(s[h], s[h + 1]):
            for d in range(T // 2 + 1):
                if T % 2 == 0 and 2 * d == T and 2 * p >= T:
                    continue
                q = (p - d) % T
                key = (min(p, q), max(p, q))
                assert key not in seen, (key, h, seen.get(key))
                seen[key] = h
        assert D.band_tiles(N, G, h) == sum(1 for v in seen.values() if v == h)
        assert D.band_computed_entries(N, G, h) == 64 * 64 * D.band_tiles(N, G, h)
    assert len(seen) == T * (T + 1) // 2
    if T >= 8 * G:
        w = [D.band_tiles(N, G, h) for h in range(G)]
        assert max(w) / min(w) < 1.2


def test_peer_band_halves_nvlink_traffic():
    N, G = 100_000, 8
    band = [D.peer_mirror_bytes(N, G, h, "band") for h in range(G)]
    tiles = [D.peer_mirror_bytes(N, G, h, "tiles") for h in range(G)]
    # 4.4 GB per rank, balanced, vs up to 9.3 GB for lower-tile ranges
    assert max(band) < 4.5e9 and max(band) / min(band) < 1.01
    assert max(tiles) > 2.0 * max(band)
    work = [D.band_computed_entries(N, G, h) for h in range(G)]
    # every pair once, plus the upper halves of the T full diagonal tiles
    assert abs(sum(work) - (N * (N + 1) // 2 + (64 * 64 - 64 * 65 // 2) * (-(-N // 64)))) < 64 * 64
    assert max(work) / (N * N / (2 * G)) < 1.005


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
