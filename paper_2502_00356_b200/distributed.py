"""Multi-GPU sharding of the hot path: one process per GPU.

Both workloads shard with NO data-path communication -- Matern entries and
BesselK elements are pure functions of their inputs -- so a rank computes its
shard from the replicated (tiny) inputs and keeps it; collectives appear only
in the optional gathers below (NCCL over NVLink on GPUs, gloo in CPU tests):

  * full matrix  -> contiguous row blocks [N g / G, N (g+1) / G): contiguous in
    row-major storage; inside its diagonal block a rank computes each pair
    once and mirrors it (bgk_matern_covariance);
  * packed lower tiles (the 160 GB N=200K layout) -> contiguous ranges of the
    tile index l = p(p+1)/2 + q; every tile is the same work, so equal counts
    are an area-balanced split;
  * BesselK batches -> contiguous 1/G slices.

The compute callables are injectable so the plumbing (shard arithmetic,
assembly, gathers) is testable on CPU with the oracle standing in for the GPU.
"""

from __future__ import annotations

import numpy as np


def row_shard(N: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of the N x N matrix owned by ``rank`` of ``world``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return N * rank // world, N * (rank + 1) // world


def row_shards(N: int, world: int) -> list[tuple[int, int]]:
    return [row_shard(N, world, g) for g in range(world)]


def tile_shard(ntiles: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous packed-lower-tile range [l0, l1) for ``rank`` (equal counts)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return ntiles * rank // world, ntiles * (rank + 1) // world


def batch_shard(n: int, world: int, rank: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def computed_entries(N: int, r0: int, r1: int) -> int:
    """Entries a row-block shard evaluates: the diagonal block once per pair,
    the rest of its rows directly ((1/G - 1/(2G^2)) N^2 each)."""
    R = r1 - r0
    return R * (N - R) + R * (R + 1) // 2


def _dist():
    import torch.distributed as dist

    return dist


def _rank_world(group=None) -> tuple[int, int]:
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def generate_covariance_sharded(locs, theta, cfg=None, *, device=None, group=None,
                                compute=None):
    """This rank's row block of the covariance matrix (no communication).

    Returns (r0, r1, block) with block = rows [r0, r1) as a tensor on ``device``
    (default: the current CUDA device).  ``compute(locs, theta, cfg, rows)`` may
    replace the GPU kernel (tests use the CPU oracle)."""
    rank, world = _rank_world(group)
    N = int(np.asarray(locs.coords if hasattr(locs, "coords") else locs).shape[0])
    r0, r1 = row_shard(N, world, rank)
    if compute is None:
        from .besselk import DEFAULT_CONFIG
        from .covariance import generate_covariance

        import torch

        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        block = generate_covariance(locs, theta, cfg or DEFAULT_CONFIG, rows=(r0, r1),
                                    device=dev).data
    else:
        block = compute(locs, theta, cfg, (r0, r1))
    return r0, r1, block


def gather_rows(block, N: int, *, dst: int = 0, group=None):
    """Assemble the full N x N matrix on rank ``dst`` from every rank's row block
    (one ``gather`` of equal-size padded blocks).  Other ranks return None."""
    import torch

    dist = _dist()
    rank, world = _rank_world(group)
    shards = row_shards(N, world)
    rmax = max(r1 - r0 for r0, r1 in shards)
    pad = torch.zeros((rmax, N), dtype=block.dtype, device=block.device)
    pad[:block.shape[0]] = block
    if world == 1:
        return block
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[:r1 - r0] for b, (r0, r1) in zip(bufs, shards)], 0)


def bessel_k_batch_sharded(x, nu, cfg=None, *, group=None, gather: bool = False,
                           compute=None):
    """BesselK over this rank's contiguous slice of (x, nu); with ``gather`` the
    full log K vector is all-gathered on every rank.  Returns (i0, i1, log_k)."""
    import torch

    dist = _dist()
    rank, world = _rank_world(group)
    n = len(x)
    i0, i1 = batch_shard(n, world, rank)
    if compute is None:
        from .besselk import DEFAULT_CONFIG, bessel_k_batch

        logk = bessel_k_batch(x[i0:i1], nu[i0:i1], cfg or DEFAULT_CONFIG, validate=False).log_value
        if not isinstance(logk, torch.Tensor):
            logk = torch.from_numpy(logk).cuda()
    else:
        logk = compute(x[i0:i1], nu[i0:i1], cfg)
    if not gather or world == 1:
        return i0, i1, logk
    sizes = [batch_shard(n, world, g) for g in range(world)]
    m = max(b - a for a, b in sizes)
    pad = torch.zeros(m, dtype=logk.dtype, device=logk.device)
    pad[:logk.numel()] = logk
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return 0, n, torch.cat([b[:e - s] for b, (s, e) in zip(bufs, sizes)])
