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


# ---------------------------------------------------------------------------------------
# fused compute + NVLink peer stores (every lower macro tile computed exactly once)
# ---------------------------------------------------------------------------------------

MACRO = 64


def macro_row_starts(N: int, world: int) -> list[int]:
    """Owner h holds macro rows [s[h], s[h+1]) (64-row blocks), as equal as possible."""
    T = -(-N // MACRO)
    return [T * g // world for g in range(world + 1)]


def owner_rows(N: int, world: int, rank: int) -> tuple[int, int]:
    s = macro_row_starts(N, world)
    return min(N, MACRO * s[rank]), min(N, MACRO * s[rank + 1])


def peer_tile_range(N: int, world: int, rank: int) -> tuple[int, int]:
    """This rank's equal share of the T(T+1)/2 lower macro tiles (equal work)."""
    T = -(-N // MACRO)
    total = T * (T + 1) // 2
    return total * rank // world, total * (rank + 1) // world


PEER_MODES = ("band", "tiles")


def band_tiles(N: int, world: int, rank: int) -> int:
    """Macro tiles rank computes in "band" mode: for each of its macro rows p the
    tiles q = p - d (mod T), d = 0 .. floor(T/2), d = T/2 (T even) only for p < T/2."""
    T = -(-N // MACRO)
    s = macro_row_starts(N, world)
    n = 0
    for p in range(s[rank], s[rank + 1]):
        n += T // 2 + 1
        if T % 2 == 0 and 2 * p >= T:
            n -= 1
    return n


def band_computed_entries(N: int, world: int, rank: int) -> int:
    """Matrix entries rank computes in "band" mode (edge tiles clipped at N)."""
    T = -(-N // MACRO)
    s = macro_row_starts(N, world)
    n = 0
    for p in range(s[rank], s[rank + 1]):
        rp = min(MACRO, N - MACRO * p)
        for d in range(T // 2 + 1):
            if T % 2 == 0 and 2 * d == T and 2 * p >= T:
                continue
            n += rp * min(MACRO, N - MACRO * ((p - d) % T))
    return n


def peer_mirror_bytes(N: int, world: int, rank: int, mode: str = "band") -> int:
    """Bytes rank stores into OTHER ranks' blocks (NVLink traffic), both modes."""
    T = -(-N // MACRO)
    s = macro_row_starts(N, world)
    own = [0] * T
    for h in range(world):
        for p in range(s[h], s[h + 1]):
            own[p] = h

    def rows(p):
        return min(MACRO, N - MACRO * p)

    total = 0
    if mode == "band":
        for p in range(s[rank], s[rank + 1]):
            for d in range(T // 2 + 1):
                if T % 2 == 0 and 2 * d == T and 2 * p >= T:
                    continue
                q = (p - d) % T
                if d and own[q] != rank:
                    total += rows(p) * rows(q) * 8
    else:
        l0, l1 = peer_tile_range(N, world, rank)
        p = 0
        for l in range(l0, l1):
            while (p + 1) * (p + 2) // 2 <= l:
                p += 1
            q = l - p * (p + 1) // 2
            b = rows(p) * rows(q) * 8
            total += b * (own[p] != rank) + (b if p != q and own[q] != rank else 0)
    return total


def _launch_peer(plan, lx, ly, N, starts, bases, l0, l1, rank=None):
    """tiles mode: lower tiles [l0, l1); band mode (rank given): rank's cyclic half band."""
    import ctypes

    import torch

    from . import _lib

    L = _lib.lib()
    G = len(bases)
    st = (ctypes.c_int64 * (G + 1))(*starts)
    bp = (ctypes.c_void_p * G)(*bases)
    stream = torch.cuda.current_stream().cuda_stream
    if rank is not None:
        rc = L.bgk_matern_covariance_peer_band(ctypes.byref(plan), lx.data_ptr(), ly.data_ptr(),
                                               N, G, st, bp, rank, stream)
        _lib.check(rc, "bgk_matern_covariance_peer_band")
        return
    rc = L.bgk_matern_covariance_peer(ctypes.byref(plan), lx.data_ptr(), ly.data_ptr(), N, G, st,
                                      bp, l0, l1, stream)
    _lib.check(rc, "bgk_matern_covariance_peer")


def generate_covariance_peer_emulated(locs, theta, world: int, cfg=None, mode: str = "band"):
    """Single-process check of the peer-store kernel: ``world`` owner buffers on the
    current GPU stand in for the ranks' HBM and every rank's share is launched
    here.  Returns the owners' row blocks (their concatenation is the full
    matrix)."""
    import torch

    from .besselk import DEFAULT_CONFIG
    from .covariance import _coords, matern_plan

    lx, ly = _coords(locs)
    N = lx.numel()
    plan = matern_plan(theta, cfg or DEFAULT_CONFIG)
    starts = macro_row_starts(N, world)
    blocks = []
    for g in range(world):
        r0, r1 = owner_rows(N, world, g)
        blocks.append(torch.empty((r1 - r0, N), dtype=torch.float64, device=lx.device))
    bases = [b.data_ptr() if b.numel() else 1 for b in blocks]
    if mode not in PEER_MODES:
        raise ValueError(f"mode must be one of {PEER_MODES}")
    for g in range(world):
        if mode == "band":
            _launch_peer(plan, lx, ly, N, starts, bases, 0, 0, rank=g)
        else:
            _launch_peer(plan, lx, ly, N, starts, bases, *peer_tile_range(N, world, g))
    return blocks


class PeerMatrix:
    """This rank's row block plus IPC mappings of every other rank's block.

    Collective construction (all ranks of ``group``): allocate the local block,
    export a CUDA IPC handle, all-gather the handles, enable peer access and map
    the peers.  ``compute`` then runs this rank's tile range of the fused kernel;
    the whole matrix is complete after ``compute`` on every rank plus a barrier.
    """

    def __init__(self, N: int, group=None, device=None, mode: str = "band"):
        import ctypes

        import torch

        from . import _lib

        dist = _dist()
        self.group = group
        self.rank, self.world = _rank_world(group)
        self.N = N
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.r0, self.r1 = owner_rows(N, self.world, self.rank)
        self.block = torch.empty((self.r1 - self.r0, N), dtype=torch.float64, device=self.device)
        L = _lib.lib()
        handle = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        off = ctypes.c_uint64()
        ptr = self.block.data_ptr() if self.block.numel() else 0
        if ptr:
            _lib.check(L.bgk_ipc_export(ptr, handle, ctypes.byref(off)), "bgk_ipc_export")
        mine = (bytes(handle.raw), int(off.value), self.device.index, bool(ptr))
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self.bases, self._opened = [], []
        err = None
        try:
            for h, (hb, o, dev, ok) in enumerate(everyone):
                if h == self.rank or not ok:
                    self.bases.append(ptr or 1)  # empty blocks are never written
                    continue
                if dev != self.device.index:
                    can = ctypes.c_int(0)
                    _lib.check(L.bgk_can_access_peer(dev, ctypes.byref(can)),
                               "bgk_can_access_peer")
                    if not can.value:
                        raise RuntimeError(f"cudaDeviceCanAccessPeer({self.device.index} -> "
                                           f"{dev}) = 0: no P2P path for the mirror stores")
                    _lib.check(L.bgk_enable_peer_access(dev), "bgk_enable_peer_access")
                p = ctypes.c_void_p()
                _lib.check(L.bgk_ipc_open(hb, o, ctypes.byref(p)), "bgk_ipc_open")
                self.bases.append(p.value)
                self._opened.append((p.value, o))
        except Exception as ex:  # noqa: BLE001 -- reported collectively below
            err = f"rank {self.rank}: {type(ex).__name__}: {ex}"
        # every rank learns whether every rank mapped every peer, so they all take the
        # peer path or all fall back together (no rank left waiting in a collective)
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)
        bad = [e for e in errs if e]
        if bad:
            self.close()
            raise RuntimeError("peer mapping failed: " + "; ".join(bad))
        self.starts = macro_row_starts(N, self.world)
        if mode not in PEER_MODES:
            raise ValueError(f"mode must be one of {PEER_MODES}")
        self.mode = mode
        self.tiles = peer_tile_range(N, self.world, self.rank)

    def compute(self, plan, lx, ly):
        """Launch this rank's tiles (stream-ordered; no barrier).  "band": the cyclic
        half band of its own macro rows (every direct store local, only mirrors
        cross NVLink); "tiles": an equal contiguous range of lower tiles."""
        if self.mode == "band":
            _launch_peer(plan, lx, ly, self.N, self.starts, self.bases, 0, 0, rank=self.rank)
        else:
            _launch_peer(plan, lx, ly, self.N, self.starts, self.bases, *self.tiles)

    def close(self):
        from . import _lib

        L = _lib.load_library()
        for p, o in self._opened:
            L.bgk_ipc_close(p, o)
        self._opened = []


def generate_covariance_peer(locs, theta, cfg=None, *, group=None, device=None, mode="band"):
    """Row block of this rank, with every lower macro tile of the matrix computed
    once across the group and transposes stored straight into the owning GPU's
    memory over NVLink.  Returns (r0, r1, block); collective."""
    import torch

    from .besselk import DEFAULT_CONFIG
    from .covariance import _coords, matern_plan

    lx, ly = _coords(locs)
    pm = PeerMatrix(lx.numel(), group=group, device=device, mode=mode)
    pm.compute(matern_plan(theta, cfg or DEFAULT_CONFIG), lx, ly)
    torch.cuda.synchronize(pm.device)
    _dist().barrier(group=group)
    pm.close()
    return pm.r0, pm.r1, pm.block
