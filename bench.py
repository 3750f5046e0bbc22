#!/usr/bin/env python
"""Benchmark: Matern covariance generation at N=100K (the metric BASELINE.json
quotes: "BesselK evals/s; Matern cov-gen time at N=100K (1/2/4/8 B200) vs CPU").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload m100|m10|m50|m200|bk|bk1m]
    torchrun --nproc-per-node N bench.py --gpus N ...    (one rank per GPU, NCCL)

One step = one generation of the whole N x N fp64 matrix, inputs resident in HBM.
N>1: fused compute + NVLink peer stores (each 64x64 tile pair computed once by one
rank, its transpose stored straight into the owner's HBM), else independent row
blocks.  Timed with CUDA events on the launching stream between a barrier +
synchronize on both sides; the job time is the MAX over ranks.  Rank 0 prints ONE
JSON line.

--impl reference runs the reference's own CPU implementation on the host cores:
the UNMODIFIED numba kernels of the reference package (baseline/_ref, driven like
the reference's caller / SPEC: oracle/ref_numba.py), or the oracle port (oracle/,
a C restatement bitwise equal to the numba kernels) when numba or the install is
missing.  Its K timed steps together run ONE whole job (step k computes the k-th
1/K of the lower tiles + their mirror, or of the BesselK batch), so `value` is a
measured whole-job time, not an extrapolation.  Under torchrun only rank 0 runs.
"""

from __future__ import annotations

import argparse
import glob
import hashlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20250201
# algorithmic FP64-pipe ops per unit (DFMA counted once) -- the
# naive-implementation work figure, reported as roofline.algorithmic_frac only
W_MATERN = {0.3: 495.0, 0.8: 497.0, 1.5: 500.0, 1.7: 501.0, 2.9: 505.0}
W_BESSELK = 700.0
E2E_WARM = 2  # untimed end-to-end calls first (page-locked buffers, host threads)
NVLINK_GBS = 770.0  # per-direction NVLink 5 bandwidth a GPU can drive (B200_PROFILING.md)

WORKLOADS = {
    "m100": dict(N=100_000, nus=[1.5], desc="Matern covariance N=100K full fp64 matrix, nu=1.5, "
                 "sigma2=1, beta=0.1"),
    "m10": dict(N=10_000, nus=[1.5], desc="Matern covariance N=10K, nu=1.5, sigma2=1, beta=0.1"),
    "m50": dict(N=50_000, nus=[0.3, 0.8, 1.7, 2.9], desc="Matern covariance N=50K, nu sweep "
                "{0.3,0.8,1.7,2.9}, one matrix per nu per step"),
    "m200": dict(N=200_000, nus=[1.5], desc="Matern covariance N=200K lower-triangle tiles "
                 "(ts=256, packed, ~160 GB), area-balanced tile shards"),
    "bk": dict(n=64 << 20, desc="BesselK batch, 64Mi random (x,nu), x in (0,140], nu in (0,20]"),
    "bk1m": dict(n=1_000_000, desc="BesselK batch, 1M random (x,nu), x in (0,140], nu in (0,20] "
                 "(BASELINE.json configs[0])"),
}


def release_host_cache():
    """Give the page-locked host memory of a finished leg back to the OS (torch caches
    freed pinned blocks; an idle 80 GB pinned block slows the next leg's host work)."""
    import gc

    import torch

    gc.collect()
    if hasattr(torch._C, "_host_emptyCache"):
        torch._C._host_emptyCache()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def src_sha16() -> str:
    """Hash of the kernel sources: ties a committed ncu summary to this build."""
    h = hashlib.sha256()
    for p in sorted(glob.glob(os.path.join(ROOT, "paper_2502_00356_b200", "csrc", "*"))):
        with open(p, "rb") as fh:
            h.update(os.path.basename(p).encode())
            h.update(fh.read())
    return h.hexdigest()[:16]


# ---------------------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------------------

class Dist:
    """One process per GPU (torchrun env).  NCCL by default; BGK_BENCH_BACKEND=gloo
    lets several ranks share one GPU (device = LOCAL_RANK mod device count) to test
    the N>1 harness on a single-GPU box."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = os.environ.get("BGK_BENCH_BACKEND", "nccl")
        self.pg = None
        self.device_index = self.local
        self.nccl_log = None

    def init(self):
        import torch

        if torch.cuda.is_available():
            self.device_index = self.local % torch.cuda.device_count()
            torch.cuda.set_device(self.device_index)
            # NCCL refuses two ranks on one GPU: when the node has fewer GPUs than
            # local ranks (a harness test on a one-GPU box), the control-plane
            # collectives (barrier, max over ranks) go over gloo instead -- the data
            # path has no collective either way
            lws = int(os.environ.get("LOCAL_WORLD_SIZE", str(self.world)))
            if (self.backend == "nccl" and "BGK_BENCH_BACKEND" not in os.environ
                    and torch.cuda.device_count() < lws):
                self.backend = "gloo"
                log(f"[bench] {lws} local ranks on {torch.cuda.device_count()} GPU(s): "
                    "gloo for barriers and reductions")
        if self.world > 1 and self.pg is None:
            import torch.distributed as dist

            if self.backend == "nccl" and self.rank == 0 and "NCCL_DEBUG" not in os.environ:
                # rank 0's communicator lines (transport, NVLS) into a file, not stdout
                fd, self.nccl_log = tempfile.mkstemp(prefix="nccl_rank0_", suffix=".log")
                os.close(fd)
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ["NCCL_DEBUG_SUBSYS"] = "INIT,GRAPH,NVLS"
                os.environ["NCCL_DEBUG_FILE"] = self.nccl_log
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(self.backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            if self.backend == "nccl":
                self.pg.barrier(device_ids=[self.device_index])
            else:
                self.pg.barrier()

    def _reduce(self, v: float, op) -> float:
        import torch

        dev = f"cuda:{self.device_index}" if self.backend == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v: float) -> float:
        return self._reduce(v, self.pg.ReduceOp.MAX) if self.pg else v

    def sum(self, v: float) -> float:
        return self._reduce(v, self.pg.ReduceOp.SUM) if self.pg else v

    def nccl_summary(self) -> dict | None:
        """Communicator lines NCCL logged on rank 0 (transport / NVLS evidence)."""
        if not self.nccl_log or not os.path.exists(self.nccl_log):
            return None
        with open(self.nccl_log, errors="replace") as fh:
            lines = [l.strip() for l in fh if l.strip()]
        keep = [l for l in lines if any(k in l for k in ("Init COMPLETE", "NVLS", "P2P", "via",
                                                         "comm 0x", "Channel 00"))]
        for l in keep[:40]:
            log("[nccl rank0]", l)
        return {"lines": len(lines), "nvls": any("NVLS" in l and "enabled" in l.lower()
                                                 for l in lines),
                "sample": keep[:8]}

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        # nvidia-smi takes a few hundred ms to start: wait for its first sample so a
        # short timed region is not over before sampling begins
        t_end = time.time() + 3.0
        while time.time() < t_end and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    smax.append(float(f[2]))
                    power.append(float(f[3]))
                except ValueError:
                    continue
                for n, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "power_w_max": max(power) if power else None, "samples": len(sm),
                "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------------------
# measured peaks (roofline denominators)
# ---------------------------------------------------------------------------------------

def measure_fp64_peak(device) -> dict:
    import ctypes

    import torch

    from paper_2502_00356_b200 import _lib

    L = _lib.lib()
    blocks = 148 * 8
    scratch = torch.empty(blocks * 256, dtype=torch.float64, device=device)
    stream = torch.cuda.current_stream()
    n = ctypes.c_double()
    best = 0.0
    for it in (64, 512, 2048, 2048):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record(stream)
        _lib.check(L.bgk_fp64_probe(scratch.data_ptr(), blocks, it, stream.cuda_stream,
                                    ctypes.byref(n)), "bgk_fp64_probe")
        e.record(stream)
        e.synchronize()
        best = max(best, n.value / (s.elapsed_time(e) * 1e-3))
    return {"fp64_pipe_ops_per_s": best,
            "how": "bgk_fp64_probe: 1184x256 threads x 8 independent DFMA chains, best of 4, "
                   "CUDA events; DFMA = 1 FP64-pipe op"}


def measure_pcie(device, nbytes=1 << 30) -> dict:
    """Pinned host <-> device copy bandwidth on this box (the e2e roofline)."""
    import torch

    n = nbytes // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device=device)
    h.fill_(1.0)
    res = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 0.0
        for _ in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(device)
            s.record()
            fn()
            e.record()
            e.synchronize()
            best = max(best, nbytes / (s.elapsed_time(e) * 1e-3) / 1e9)
        res[f"{name}_gbs"] = best
    res["how"] = f"pinned {nbytes >> 20} MiB copy_, best of 4, CUDA events"
    del h, d
    release_host_cache()
    return res


# ---------------------------------------------------------------------------------------
# CPU reference (the reference package's numba kernels, or the oracle port)
# ---------------------------------------------------------------------------------------

def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # noqa: PLC0415

    return oracle


def _ref_numba():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_numba  # noqa: PLC0415

    return ref_numba


class CpuMaternJob:
    """The restated generate_covariance of one matrix (lower tiles ts=256 + mirror)
    on the host cores, runnable in lower-tile slices: the reference's numba
    matern_tile (kind "reference") or the oracle port (kind "port")."""

    def __init__(self, locs, nu, threads, kind, out):
        self.kind, self.locs, self.nu, self.threads, self.out = kind, locs, nu, threads, out
        N = locs.shape[0]
        T = -(-N // 256)
        self.ntiles = T * (T + 1) // 2
        if kind == "reference":
            self.job = _ref_numba().CovarianceJob(locs, 1.0, 0.1, nu, out, threads)
        else:
            self.orc = _oracle()
            self.lx = np.ascontiguousarray(locs[:, 0])
            self.ly = np.ascontiguousarray(locs[:, 1])

    def run(self, l0, l1):
        if self.kind == "reference":
            self.job.run(l0, l1)
        else:
            self.orc.generate_covariance_tiles(self.lx, self.ly, 1.0, 0.1, self.nu, self.out,
                                               l0, l1, threads=self.threads)

    def close(self):
        if self.kind == "reference":
            self.job.close()


def cpu_kind() -> str:
    return "reference" if _ref_numba().available() else "port"


def touch_host(a, threads):
    _oracle().touch(a.reshape(-1), threads)


def cpu_matern_sample(N, nu, locs, target_s=12.0, kind=None) -> dict:
    """Bounded sample for our arm's cpu_baseline: the restated generate_covariance
    of the first n_s locations (a principal submatrix of the same job, lower tiles
    + mirror), grown until it takes ~target_s, scaled to N(N+1)/2 entries."""
    threads = cpu_threads()
    kind = kind or cpu_kind()
    ns = 2048
    while True:
        out = np.empty((ns, ns))
        touch_host(out, threads)
        job = CpuMaternJob(locs[:ns], nu, threads, kind, out)
        if kind == "reference":
            job.run(0, 1)  # numba JIT outside the timing
        t0 = time.perf_counter()
        job.run(0, job.ntiles)
        t = time.perf_counter() - t0
        job.close()
        del out
        if t >= target_s / 3 or ns >= N:
            break
        ns = min(N, int(ns * max(1.4, min(4.0, ((target_s / 3) / max(t, 1e-3)) ** 0.5))))
    entries = ns * (ns + 1) / 2
    rate = entries / t
    full = N * (N + 1) / 2 / rate
    return {"rate_entries_per_s": rate, "full_job_s": full, "threads": threads, "kind": kind,
            "sample": f"restated generate_covariance (lower tiles ts=256 + mirror) of the first "
                      f"{ns} of the N={N} locations, nu={nu}: {entries:.4g} computed entries in "
                      f"{t:.2f} s on {threads} threads ({'reference numba matern_tile' if kind == 'reference' else 'oracle port'}); "
                      f"scaled to N(N+1)/2 = {N * (N + 1) / 2:.4g} entries"}


def cpu_besselk_rate(x, nu, threads, kind) -> float:
    if kind == "reference":
        _ref_numba().refined_log_bessel_batch(x, nu, threads)
    else:
        _oracle().refined_log_bessel_batch(x, nu, threads=threads)


def cpu_besselk_sample(x, nu, target_s=8.0, kind=None) -> dict:
    threads = cpu_threads()
    kind = kind or cpu_kind()
    cpu_besselk_rate(x[:4096], nu[:4096], threads, kind)  # JIT / warm
    n = 1 << 18
    while True:
        t0 = time.perf_counter()
        cpu_besselk_rate(x[:n], nu[:n], threads, kind)
        t = time.perf_counter() - t0
        if t >= target_s / 4 or n >= x.size:
            break
        n = min(x.size, int(n * max(2.0, (target_s / 4) / max(t, 1e-3))))
    return {"rate": n / t, "threads": threads, "n": n, "t": t, "kind": kind}


def scalar_call_us(fn, points, calls=4000) -> float:
    """Median over points of the mean wall time per call (after a warm-up)."""
    per = []
    for x, nu in points:
        for _ in range(200):
            fn(x, nu)
        t0 = time.perf_counter()
        for _ in range(calls):
            fn(x, nu)
        per.append((time.perf_counter() - t0) / calls * 1e6)
    return statistics.median(per)


SCALAR_POINTS = [(0.05, 1.5), (2.0, 1.5), (30.0, 10.0)]


def reference_scalar_us() -> float | None:
    R = _ref_numba()
    if not R.available():
        return None
    import besselgp  # noqa: PLC0415  (baseline/_ref, put on sys.path by ref_numba)

    return scalar_call_us(lambda x, nu: besselgp.bessel_k(besselgp.EvalPoint(x, nu)),
                          SCALAR_POINTS)


# ---------------------------------------------------------------------------------------
# workloads (ours)
# ---------------------------------------------------------------------------------------

def make_locs(N):
    return np.random.default_rng(SEED).random((N, 2))


def make_bk(n):
    rng = np.random.default_rng(SEED)
    return 140.0 * (1.0 - rng.random(n)), 20.0 * (1.0 - rng.random(n))


def matern_config(workload, wl) -> dict:
    """The config dict both arms print (identical keys and values)."""
    return {"workload": f"{workload}: {wl['desc']}", "N": wl["N"], "nu": wl["nus"],
            "sigma2": 1.0, "beta": 0.1, "bins": 40, "t_window": [0.0, 9.0], "tile_size": 256,
            "layout": "packed lower tiles" if workload == "m200" else "full row-major",
            "l2": "output (0.8-160 GB) >> 126 MB L2; every step rewrites it"}


def bk_config(workload, wl) -> dict:
    return {"workload": f"{workload}: {wl['desc']}", "n": wl["n"], "bins": 40,
            "t_window": [0.0, 9.0], "small_x_threshold": 0.1,
            "l2": "inputs + outputs 24 B/element; 64Mi = 1.6 GB >> L2 (1M: 24 MB, fits L2)"}


def select_peer(args, D, N, dev):
    """N>1 full matrix: the fused peer path when every rank can map every peer, else
    independent row blocks (decided collectively).  Returns (PeerMatrix | None,
    mode, fallback_reason)."""
    if D.world == 1 or args.mode == "rows":
        return None, "rows", None if D.world == 1 else "--mode rows"
    from paper_2502_00356_b200.distributed import PeerMatrix

    try:
        pm = PeerMatrix(N, device=dev, mode=args.peer_layout)
        return pm, "peer", None
    except Exception as ex:  # noqa: BLE001 -- PeerMatrix fails on every rank together
        reason = f"{type(ex).__name__}: {ex}"
        log(f"peer mapping unavailable ({reason}); using independent row blocks")
        if args.mode == "peer":
            raise
        return None, "rows", reason




def run_matern(args, D: Dist) -> dict:
    import torch

    import paper_2502_00356_b200 as bg
    from paper_2502_00356_b200 import _lib
    from paper_2502_00356_b200.covariance import _cov_launch, _lower_launch, matern_plan
    from paper_2502_00356_b200.distributed import (band_computed_entries, computed_entries,
                                                   peer_mirror_bytes, peer_tile_range,
                                                   row_shard, tile_shard)

    wl = WORKLOADS[args.workload]
    N = wl["N"]
    nus = wl["nus"]
    dev = torch.device("cuda", D.device_index)
    locs = make_locs(N)
    lxy = torch.from_numpy(np.ascontiguousarray(locs.T)).to(dev)
    lx, ly = lxy[0], lxy[1]
    cfg = bg.DEFAULT_CONFIG
    plans = [matern_plan(bg.MaternParams(1.0, 0.1, nu), cfg) for nu in nus]
    packed = args.workload == "m200"
    ts = 256
    pm, mode, reason = (None, "packed", None) if packed else select_peer(args, D, N, dev)
    mirror_bytes = 0.0
    if packed:
        ntiles = bg.lower_tile_count(N, ts)
        l0, l1 = tile_shard(ntiles, D.world, D.rank)
        out = torch.empty((l1 - l0, ts, ts), dtype=torch.float64, device=dev)
        computed_local = float((l1 - l0) * ts * ts)  # diagonal tiles are stored complete
        stored_local = computed_local
    else:
        if pm is not None:
            r0, r1, out = pm.r0, pm.r1, pm.block
            mirror_bytes = float(peer_mirror_bytes(N, D.world, D.rank, pm.mode))
            if pm.mode == "band":
                computed_local = float(band_computed_entries(N, D.world, D.rank))
            else:
                from paper_2502_00356_b200.distributed import MACRO

                lt = np.arange(*peer_tile_range(N, D.world, D.rank), dtype=np.int64)
                pp = ((np.sqrt(8.0 * lt + 1.0) - 1.0) // 2).astype(np.int64)
                pp += ((pp + 1) * (pp + 2) // 2 <= lt)
                pp -= (pp * (pp + 1) // 2 > lt)
                qq = lt - pp * (pp + 1) // 2
                computed_local = float(np.sum(np.minimum(MACRO, N - MACRO * pp) *
                                              np.minimum(MACRO, N - MACRO * qq)))
        else:
            r0, r1 = row_shard(N, D.world, D.rank)
            out = torch.empty((r1 - r0, N), dtype=torch.float64, device=dev)
            computed_local = float(computed_entries(N, r0, r1))
        stored_local = float((r1 - r0) * N)
    stream = torch.cuda.current_stream(dev)

    def step():
        for plan in plans:
            if packed:
                _lower_launch(plan, lx, ly, N, ts, l0, l1, out)
            elif pm is not None:
                pm.compute(plan, lx, ly)
            else:
                _cov_launch(plan, lx, ly, N, r0, r1, out, N, _lib.LAYOUT_ROW_MAJOR)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    D.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(D.device_index)
    if D.rank == 0:
        clocks.start()
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    end.record(stream)
    torch.cuda.synchronize(dev)
    launches = _lib.launch_count() - launches0
    D.barrier()
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if D.rank == 0 else None
    local_ms = start.elapsed_time(end) / args.steps
    kern_ms = statistics.median(s.elapsed_time(e) for s, e in ev) / len(plans)
    ms = D.max(local_ms)
    computed = D.sum(computed_local)
    stored = D.sum(stored_local)
    res = {"ms_per_step": ms, "launches": int(D.sum(float(launches))), "clocks": clk,
           "computed_entries": computed, "stored_entries": stored, "kernel_ms": kern_ms,
           "kernel_ms_max": D.max(kern_ms), "computed_local": computed_local,
           "stored_local": stored_local, "N": N, "nus": nus, "mode": mode,
           "fallback_reason": reason, "mirror_bytes_local": mirror_bytes,
           "mirror_bytes_max": D.max(mirror_bytes), "mirror_bytes_total": D.sum(mirror_bytes)}
    # sanity: symmetry of a probe block + diagonal == sigma^2 (cheap, outside timing)
    if not packed and r1 - r0 >= 64:
        blk = out[:64, r0:r0 + 64]
        res["check_symmetric_diag_block"] = bool(torch.equal(blk, blk.T)) and bool(
            (torch.diagonal(blk) == 1.0).all())
    # ---- e2e with host buffers -------------------------------------------------------
    if not args.no_e2e and pm is not None:
        # fused peer path: H2D of the locations, the kernel, barrier, D2H of this rank's rows
        host = bg.empty_host_matrix(r1 - r0, N)
        host_t = torch.from_numpy(host)
        ts_ = []
        for k in range(E2E_WARM + max(1, min(args.steps, args.e2e_steps))):
            D.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            lxy2 = torch.from_numpy(np.ascontiguousarray(locs.T)).to(dev)
            for plan in plans:
                pm.compute(plan, lxy2[0], lxy2[1])
            torch.cuda.synchronize(dev)
            D.barrier()
            host_t.copy_(out)
            dt = time.perf_counter() - t0
            v = D.max(dt)
            if k >= E2E_WARM:
                ts_.append(v)
        res["e2e_s"] = statistics.median(ts_)
        res["e2e_h2d"] = float(locs.nbytes) * D.world
        res["e2e_d2h"] = stored * 8.0
        res["e2e_how"] = ("fused peer kernel per rank (locations H2D each step), barrier, "
                          "D2H of the rank's rows into pinned host memory; wall clock, max over ranks")
        del host, host_t
        release_host_cache()
    if pm is not None:
        D.barrier()
        pm.close()
    del out
    torch.cuda.empty_cache()

    # ---- e2e through the public API with host buffers ---------------------------------
    if not args.no_e2e and not packed and pm is None:
        host = bg.empty_host_matrix(r1 - r0, N)
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        ts_ = []
        for k in range(E2E_WARM + e2e_steps):
            D.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for nu in nus:
                bg.generate_covariance(locs, bg.MaternParams(1.0, 0.1, nu), cfg, rows=(r0, r1),
                                       out=host)  # H2D locs, device blocks, D2H rows
            torch.cuda.synchronize(dev)
            dt = time.perf_counter() - t0
            v = D.max(dt)
            if k >= E2E_WARM:
                ts_.append(v)
        res["e2e_s"] = statistics.median(ts_)
        res["e2e_h2d"] = float(locs.nbytes) * D.world * len(nus)
        from paper_2502_00356_b200.covariance import _host_threads, host_d2h_bytes

        res["e2e_d2h"] = float(host_d2h_bytes(N, (r0, r1))) * len(nus)
        if r0 == 0 and r1 == N and res["e2e_d2h"] < stored * 8.0 * len(nus):
            res["e2e_how"] = (
                "paper_2502_00356_b200.generate_covariance(numpy locs, theta, out=pinned host "
                "array): H2D of the locations; per 1 GB row block the device computes the lower "
                f"part, a 2D copy moves it (half the matrix over PCIe) and {max(1, _host_threads() * 3 // 4)} "
                "host threads mirror it into the upper triangle (non-temporal stores) while the "
                "next block computes and copies; wall clock")
        else:
            res["e2e_how"] = ("paper_2502_00356_b200.generate_covariance(numpy locs, theta, "
                              "rows=shard, out=pinned host array): H2D of the locations, device "
                              "row blocks, D2H of every row (wall clock, max over ranks)")
        del host
        release_host_cache()
    return res


def run_besselk(args, D: Dist, workload: str, steps: int, warmup: int) -> dict:
    import torch

    import paper_2502_00356_b200 as bg
    from paper_2502_00356_b200 import _lib
    from paper_2502_00356_b200.besselk import _launch_besselk
    from paper_2502_00356_b200.distributed import batch_shard

    n_total = WORKLOADS[workload]["n"]
    dev = torch.device("cuda", D.device_index)
    i0, i1 = batch_shard(n_total, D.world, D.rank)
    x, nu = make_bk(n_total)
    xd = torch.from_numpy(x[i0:i1]).to(dev)
    nd = torch.from_numpy(nu[i0:i1]).to(dev)
    stream = torch.cuda.current_stream(dev)
    cfg = bg.DEFAULT_CONFIG
    # every step rewrites its own output buffers (allocated once: no allocator work inside
    # the timed region); 64Mi: 1.6 GB of traffic per step >> L2
    outs = [torch.empty_like(xd), torch.empty_like(xd)]

    import ctypes

    c = cfg.to_c()
    L = _lib.lib()
    argv = (xd.data_ptr(), nd.data_ptr(), xd.numel(), ctypes.byref(c), _lib.ROUTE_HYBRID,
            outs[0].data_ptr(), outs[1].data_ptr(), None, stream.cuda_stream)

    def step():
        _lib.check(L.bgk_besselk_batch(*argv), "bgk_besselk_batch")

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    D.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(D.device_index)
    if D.rank == 0:
        clocks.start()
    l0 = _lib.launch_count()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        step()
    e.record(stream)
    torch.cuda.synchronize(dev)
    launches = _lib.launch_count() - l0
    clk = clocks.stop() if D.rank == 0 else None
    D.barrier()
    ms = D.max(s.elapsed_time(e) / steps)
    res = {"ms_per_step": ms, "n": n_total, "launches": int(D.sum(float(launches))), "x": x,
           "nu": nu, "clocks": clk, "steps": steps, "warmup": warmup}
    # e2e: public API with host numpy arrays (H2D x, nu; D2H log K, K and path)
    if not args.no_e2e:
        def call():
            D.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            bg.bessel_k_batch(x[i0:i1], nu[i0:i1], cfg)  # the public API, validation included
            torch.cuda.synchronize(dev)
            return D.max(time.perf_counter() - t0)

        # the host settles over the first calls (page-locked allocations; after a
        # large page-locked buffer elsewhere in the process or a test run, for
        # seconds): warm up until two consecutive calls are within 25% of the best
        # so far (at most 40 calls / 20 s), then the median of the timed calls
        best, ok, warm_calls, w0 = float("inf"), 0, 0, time.perf_counter()
        while warm_calls < E2E_WARM + 2 or (ok < 2 and warm_calls < 40
                                            and time.perf_counter() - w0 < 20.0):
            dt = call()
            warm_calls += 1
            best = min(best, dt)
            ok = ok + 1 if dt <= 1.25 * best else 0
        tt = [call() for _ in range(max(3, min(steps, args.e2e_steps + 2)))]
        res["e2e_s"] = statistics.median(tt)
        res["e2e_warm_calls"] = warm_calls
    return res


# ---------------------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------------------

def peaks_file() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def ncu_summary(kernel: str) -> dict:
    """The committed ncu summary of a kernel (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            return json.load(fh).get(kernel, {})
    except (OSError, ValueError):
        return {}


def roofline(kernel: str, workload: str, units: float, launch_s: float, p64: float, W: float,
             stored_bytes: float | None, hbm: float) -> dict:
    """The dominant kernel's roofline.  frac: EXECUTED FP64-pipe ops per unit (from the
    committed ncu capture of this build) x units / launch time / measured FP64 peak;
    algorithmic_frac: SURVEY 8(d)'s naive-algorithm W instead (above 1: the kernel
    executes fewer ops than W)."""
    s = ncu_summary(kernel)
    ops = s.get("fp64_ops_per_unit")
    d = {"bound": "fp64", "kernel": f"bgk::{kernel}", "unit": "TFLOP/s",
         "peak": p64 / 1e12,
         "op_convention": "FP64-pipe lane-ops per second (DFMA = 1 op), peak = measured "
                          "bgk_fp64_probe",
         "units_per_launch": units, "launch_ms": launch_s * 1e3}
    if ops:
        d["achieved"] = ops * units / launch_s / 1e12
        d["frac"] = ops * units / launch_s / p64
        d["executed_fp64_ops_per_unit"] = ops
        d["thread_instructions_per_unit"] = s.get("thread_inst_per_unit")
        d["issue_active"] = s.get("issue_active_pct", 0) / 100.0 or None
        d["ncu_fp64_pipe_frac"] = s.get("fp64_pipe_pct", 0) / 100.0 or None
        d["ncu_capture"] = s.get("capture")
        d["ncu_src_sha16"] = s.get("src_sha16")
        d["ncu_matches_build"] = s.get("src_sha16") == src_sha16()
    else:
        d["achieved"] = None
        d["frac"] = None
    d["algorithmic_w_per_unit"] = W
    d["algorithmic_frac"] = W * units / launch_s / p64
    d["traffic"] = (s.get("traffic") or {}).get(workload)
    if stored_bytes is not None:
        d["hbm_write_gbs"] = stored_bytes / launch_s / 1e9
        d["hbm_write_frac"] = stored_bytes / launch_s / 1e9 / hbm
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="m100")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--peer-layout", choices=["band", "tiles"], default="band",
                    help="peer mode work split: each rank's cyclic half band of its own rows "
                         "(direct stores local, mirrors over NVLink) or equal lower-tile ranges")
    ap.add_argument("--mode", choices=["auto", "peer", "rows"], default="auto",
                    help="N>1 full-matrix sharding: fused P2P mirror stores (peer) or "
                         "independent row blocks (rows); auto = peer with fallback")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=12.0,
                    help="seconds of CPU work for our arm's cpu_baseline sample")
    ap.add_argument("--ref-kind", choices=["auto", "reference", "port"], default="auto",
                    help="reference arm: the reference's numba kernels or the oracle port")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to the contract minimum of 3")
        args.warmup = 3

    D = Dist()
    wl = WORKLOADS[args.workload]
    matern = "N" in wl

    if args.impl == "reference":
        if D.rank != 0:
            return
        print(json.dumps(reference_line(args, D.world, wl, matern)), flush=True)
        return

    D.init()
    import torch

    dev = torch.device("cuda", D.device_index)
    peaks = peaks_file()
    fp64 = measure_fp64_peak(dev) if D.rank == 0 else None
    pcie = measure_pcie(dev) if D.rank == 0 else None

    # secondary: the BK batch lines, single GPU only.  They run FIRST: after the M100
    # leg's 80 GB page-locked host buffer the host needs seconds to settle, which would
    # otherwise land in the BK end-to-end calls.
    sec = {}
    if matern and not args.no_secondary and D.world == 1:
        sec["bk"] = run_besselk(args, D, "bk", 10, 3)
        sec["bk1m"] = run_besselk(args, D, "bk1m", 200, 20)
        torch.cuda.empty_cache()

    if matern:
        r = run_matern(args, D)
    else:
        r = run_besselk(args, D, args.workload, args.steps, args.warmup)

    scalar = None
    if D.rank == 0 and D.world == 1 and not args.no_secondary:
        import paper_2502_00356_b200 as bg

        ours = scalar_call_us(lambda x, nu: bg.bessel_k(bg.EvalPoint(x, nu)), SCALAR_POINTS)
        try:
            ref = reference_scalar_us()
        except Exception as ex:  # noqa: BLE001
            log(f"reference scalar timing unavailable: {ex}")
            ref = None
        scalar = {"metric": "bessel_k(EvalPoint) latency", "value": ours, "unit": "us/call",
                  "reference_us": ref,
                  "points": SCALAR_POINTS,
                  "how": "mean over 4000 calls per point after 200 warm, median over points; "
                         "ours: one launch + one sync through bgk_besselk_scalar (mapped "
                         "page-locked slot); reference: besselgp.bessel_k from baseline/_ref "
                         "(numba), same process"}

    nccl = D.nccl_summary() if D.rank == 0 else None
    if D.rank == 0:
        line = build_line(args, D.world, wl, matern, r, sec, peaks, fp64, pcie, scalar, nccl)
        if D.world > 1:
            line["control_backend"] = D.backend  # barriers / max over ranks (no data-path collective)
        print(json.dumps(line), flush=True)
    D.barrier()
    D.close()


def bk_line(r, world, p64, workload) -> dict:
    n = r["n"]
    t = r["ms_per_step"] * 1e-3
    wl = WORKLOADS[workload]
    d = {"metric": "BesselK evals/s", "value": n / t, "unit": "evals/s",
         "ms_per_step": r["ms_per_step"], "steps": r["steps"], "warmup": r["warmup"],
         "config": bk_config(workload, wl),
         "roofline": roofline("besselk_kernel", workload, n / world, t, p64, W_BESSELK,
                              None, 0.0)}
    if "e2e_s" in r:
        d["e2e"] = {"value": n / r["e2e_s"], "unit": "evals/s",
                    "h2d_bytes_per_step": 16.0 * n, "d2h_bytes_per_step": 17.0 * n,
                    "how": "bessel_k_batch(numpy x, numpy nu): validation, H2D, kernel, D2H of "
                           "log K, K and path (wall clock); median of the timed calls after "
                           f"{r.get('e2e_warm_calls')} warm-up calls (until two consecutive "
                           "calls are within 25% of the best)"}
    return d


def build_line(args, world, wl, matern, r, sec, peaks, fp64, pcie, scalar, nccl):
    hbm = peaks.get("hbm_gbs", 6547.5)
    p64 = fp64["fp64_pipe_ops_per_s"]
    nominal = 148 * 64 * 1.965e9
    if matern:
        N = r["N"]
        nus = r["nus"]
        W = statistics.mean(W_MATERN.get(nu, 500.0) for nu in nus)
        t = r["ms_per_step"] * 1e-3
        workload = args.workload
        metric = "Matern cov-gen time at N=100K" if workload == "m100" else \
            f"Matern cov-gen time ({wl['desc']})"
        execution = (f"packed lower-tile shards x{world}" if workload == "m200" else
                     f"fused compute + NVLink P2P mirror stores x{world}: each 64x64 tile pair "
                     f"computed once ({args.peer_layout} layout)" if r.get("mode") == "peer"
                     else f"row-block shards x{world}, no collective")
        line = {
            "metric": metric,
            "value": t,
            "unit": "s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"],
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: rng(20250201).random((N,2)) unit-square locations",
            "config": matern_config(workload, wl),
            "execution": execution,
            "mode": r.get("mode"),
            "entries_per_s": r["stored_entries"] * len(nus) / t,
            "computed_entries_per_s": r["computed_entries"] * len(nus) / t,
            "roofline": roofline("matern_kernel", workload, r["computed_local"],
                                 r["kernel_ms"] * 1e-3, p64, W, r["stored_local"] * 8.0, hbm),
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
        }
        line["roofline"]["peak_source"] = fp64["how"] + f" (nominal 148x64x1.965GHz = {nominal / 1e12:.2f})"
        if r.get("fallback_reason"):
            line["fallback_reason"] = r["fallback_reason"]
        if world > 1 and r.get("mode") == "peer":
            kt = r["kernel_ms_max"] * 1e-3
            line["nvlink"] = {"mirror_bytes_per_rank_max": r["mirror_bytes_max"],
                              "mirror_bytes_total": r["mirror_bytes_total"],
                              "achieved_gbs_per_rank_max": r["mirror_bytes_max"] / kt / 1e9,
                              "frac_of_nvlink": r["mirror_bytes_max"] / kt / 1e9 / NVLINK_GBS,
                              "nvlink_gbs": NVLINK_GBS,
                              "how": "P2P mirror stores from the kernel's store phase into "
                                     "peers' CUDA-IPC-mapped blocks; bytes from "
                                     "distributed.peer_mirror_bytes, over the rank's kernel time"}
        if nccl is not None:
            line["nccl"] = nccl
        if "check_symmetric_diag_block" in r:
            line["check_symmetric_diag_block"] = r["check_symmetric_diag_block"]
        if "e2e_s" in r:
            moved = r["e2e_h2d"] + r["e2e_d2h"]
            line["e2e"] = {"value": r["e2e_s"], "unit": "s", "h2d_bytes_per_step": r["e2e_h2d"],
                           "d2h_bytes_per_step": r["e2e_d2h"], "how": r["e2e_how"]}
            if pcie:
                line["e2e"]["pcie"] = {"achieved_gbs": moved / r["e2e_s"] / 1e9,
                                       "peak_d2h_gbs": pcie["d2h_gbs"],
                                       "peak_h2d_gbs": pcie["h2d_gbs"],
                                       "frac": moved / r["e2e_s"] / 1e9 / pcie["d2h_gbs"],
                                       "how": pcie["how"] + "; frac = bytes moved / e2e time / "
                                              "measured D2H peak (D2H dominates)"}
        if world == 1 and not args.no_cpu_baseline:
            c = cpu_matern_sample(N, nus[0], make_locs(N), target_s=args.cpu_sample_s)
            line["cpu_baseline"] = {"value": c["full_job_s"] * len(nus), "unit": "s",
                                    "cores": c["threads"], "kind": c["kind"],
                                    "sample": c["sample"], "cpu": cpu_model()}
    else:
        line = {"n_gpus": world, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: x=140(1-U), nu=20(1-V), rng(20250201)",
                "gpu_launches": r["launches"], "clocks": r["clocks"]}
        line.update(bk_line(r, world, p64, args.workload))
        if world == 1 and not args.no_cpu_baseline:
            c = cpu_besselk_sample(r["x"], r["nu"], target_s=args.cpu_sample_s * 2 / 3)
            line["cpu_baseline"] = {"value": c["rate"], "unit": "evals/s", "cores": c["threads"],
                                    "kind": c["kind"], "sample": f"first {c['n']} elements, "
                                    f"{c['t']:.2f} s", "cpu": cpu_model()}
    secondary = []
    for name, s in sec.items():
        d = bk_line(s, 1, p64, name)
        if not args.no_cpu_baseline and name == "bk1m":
            c = cpu_besselk_sample(s["x"], s["nu"], target_s=args.cpu_sample_s * 2 / 3)
            d["cpu_baseline"] = {"value": c["rate"], "unit": "evals/s", "cores": c["threads"],
                                 "kind": c["kind"],
                                 "sample": f"first {c['n']} elements of the same batch, "
                                           f"{c['t']:.2f} s"}
        secondary.append(d)
    if scalar is not None:
        secondary.append(scalar)
    if secondary:
        line["secondary"] = secondary
    line["fp64_peak_measured_tops"] = p64 / 1e12
    if pcie:
        line["pcie_measured"] = pcie
    line["src_sha16"] = src_sha16()
    return line


# ---------------------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------------------

def reference_line(args, world, wl, matern) -> dict:
    """The reference's CPU implementation on all host cores.  The K timed steps
    together run ONE whole job: step k = the k-th 1/K of the lower tiles (+ mirror)
    of every matrix, or of the BesselK batch; the W warm-up steps run small slices
    (numba JIT, thread pool, page faults) outside the timing."""
    threads = cpu_threads()
    if args.ref_kind == "auto":
        kind = cpu_kind()
    else:
        kind = args.ref_kind
    why = None if kind == "reference" else _ref_numba().unavailable_reason()
    K, W = args.steps, args.warmup
    common = {"impl": "reference", "n_gpus": world, "steps": K, "warmup": W,
              "scaling": "strong", "vs_baseline": None, "dtype": "f64"}
    if matern and args.workload != "m200":
        N = wl["N"]
        nus = wl["nus"]
        locs = make_locs(N)
        t_alloc = time.perf_counter()
        out = np.empty((N, N))
        touch_host(out, threads)  # first touch outside the timed steps
        t_alloc = time.perf_counter() - t_alloc
        jobs = [CpuMaternJob(locs, nu, threads, kind, out) for nu in nus]
        L = jobs[0].ntiles
        edges = [L * k // K for k in range(K + 1)]
        for w in range(W):  # small slices: JIT, pool start-up
            for job in jobs:
                job.run(0, max(1, L // (100 * K)))
        step_s = []
        for k in range(K):
            t0 = time.perf_counter()
            for job in jobs:
                job.run(edges[k], edges[k + 1])
            step_s.append(time.perf_counter() - t0)
        total = sum(step_s)
        # the whole matrix exists now: spot-check symmetry and the diagonal
        ok = bool(np.array_equal(out[:256, :256], out[:256, :256].T)) and bool(
            (np.diagonal(out)[:1000] == 1.0).all())
        # the port (and the reference, if it ran) on the same slice for comparison
        comp = {}
        if len(nus) == 1:
            sl = (edges[0], edges[1])
            for kd in (["reference", "port"] if kind == "reference" else ["port"]):
                j = jobs[0] if kd == kind else CpuMaternJob(locs, nus[0], threads, kd, out)
                t0 = time.perf_counter()
                j.run(*sl)
                comp[kd + "_s"] = time.perf_counter() - t0
                if j is not jobs[0]:
                    j.close()
            comp["slice"] = f"lower tiles [{sl[0]}, {sl[1]}) of {L} (+ mirror)"
        for job in jobs:
            job.close()
        del out
        impl = ("the reference package's numba kernels.matern_tile (baseline/_ref), restated "
                "caller SPEC.md:324-332" if kind == "reference" else
                "oracle port (C restatement of kernels.matern_tile, bitwise equal to numba)")
        line = dict(common)
        line.update({
            "metric": "Matern cov-gen time at N=100K" if args.workload == "m100"
            else f"Matern cov-gen time ({wl['desc']})",
            "value": total, "unit": "s", "ms_per_step": total / K * 1e3,
            "higher_is_better": False,
            "data": "synthetic: rng(20250201).random((N,2)) unit-square locations",
            "config": matern_config(args.workload, wl),
            "execution": f"{impl}; {threads} host threads; the {K} timed steps together "
                         f"generate the whole matrix once (lower tiles ts=256 + mirror), step "
                         f"times summed",
            "step_s": step_s, "whole_job_measured": True, "check_symmetric": ok,
            "host_alloc_touch_s": t_alloc,
            "cpu_baseline": {"value": total, "unit": "s", "cores": threads, "kind": kind,
                             "sample": f"the whole job over {K} steps (not extrapolated)",
                             "cpu": cpu_model()},
            "e2e": {"value": total, "unit": "s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}})
        if comp:
            line["port_vs_reference"] = comp
    elif matern:  # m200: 160 GB of lower tiles does not fit the host; sampled + scaled
        N = wl["N"]
        c = cpu_matern_sample(N, wl["nus"][0], make_locs(N), target_s=args.cpu_sample_s, kind=kind)
        line = dict(common)
        line.update({"metric": f"Matern cov-gen time ({wl['desc']})", "value": c["full_job_s"],
                     "unit": "s", "ms_per_step": c["full_job_s"] / K * 1e3,
                     "higher_is_better": False, "data": "synthetic",
                     "config": matern_config(args.workload, wl), "whole_job_measured": False,
                     "cpu_baseline": {"value": c["full_job_s"], "unit": "s",
                                      "cores": c["threads"], "kind": kind, "sample": c["sample"],
                                      "cpu": cpu_model()},
                     "e2e": {"value": c["full_job_s"], "unit": "s", "h2d_bytes_per_step": 0,
                             "d2h_bytes_per_step": 0}})
    else:
        n = wl["n"]
        x, nu = make_bk(n)
        edges = [n * k // K for k in range(K + 1)]
        for _ in range(W):
            cpu_besselk_rate(x[:max(4096, n // (100 * K))], nu[:max(4096, n // (100 * K))],
                             threads, kind)
        step_s = []
        for k in range(K):
            t0 = time.perf_counter()
            cpu_besselk_rate(x[edges[k]:edges[k + 1]], nu[edges[k]:edges[k + 1]], threads, kind)
            step_s.append(time.perf_counter() - t0)
        total = sum(step_s)
        v = n / total
        line = dict(common)
        line.update({"metric": "BesselK evals/s", "value": v, "unit": "evals/s",
                     "ms_per_step": total / K * 1e3, "higher_is_better": True,
                     "data": "synthetic: x=140(1-U), nu=20(1-V), rng(20250201)",
                     "config": bk_config(args.workload, wl), "step_s": step_s,
                     "whole_job_measured": True,
                     "execution": ("numba loop over the reference's kernels.refined_log_bessel "
                                   "in 256 chunks on a thread pool (oracle.py:211-213 idiom)"
                                   if kind == "reference" else "oracle port, threaded") +
                                  f"; {threads} threads; the {K} steps together evaluate the "
                                  f"whole batch once",
                     "cpu_baseline": {"value": v, "unit": "evals/s", "cores": threads,
                                      "kind": kind, "sample": f"the whole {n}-element batch "
                                      f"over {K} steps", "cpu": cpu_model()},
                     "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0,
                             "d2h_bytes_per_step": 0}})
    if why:
        line["reference_unavailable"] = why
    if kind == "reference":
        try:
            line["scalar_call_us"] = reference_scalar_us()
        except Exception as ex:  # noqa: BLE001
            log(f"scalar timing failed: {ex}")
    return line


if __name__ == "__main__":
    main()
