#!/usr/bin/env python
"""Benchmark: Matern covariance generation at N=100K (the metric BASELINE.json
quotes: "BesselK evals/s; Matern cov-gen time at N=100K (1/2/4/8 B200) vs CPU").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload m100|m10|m50|m200|bk]
    torchrun --nproc-per-node N bench.py --gpus N ...    (one rank per GPU, NCCL)

One step = one generation of the whole N x N fp64 matrix (row-block shard per
rank, no data-path collective -> "scaling": "strong", total work fixed), inputs
resident in HBM.  Timed with CUDA events on the launching stream between a
barrier + synchronize on both sides; the job time is the MAX over ranks.
Rank 0 prints ONE JSON line.

--impl reference times the reference's CPU algorithm on the host cores: the
oracle port (oracle/, a C restatement of kernels.py that is bitwise equal to
the numba reference, tests/test_oracle_golden.py) on a bounded row-block
sample, extrapolated to the full job.  Under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20250201
# algorithmic FP64-pipe ops per unit (DFMA counted once)
W_MATERN = {0.3: 495.0, 0.8: 497.0, 1.5: 500.0, 1.7: 501.0, 2.9: 505.0}
W_BESSELK = 700.0
E2E_WARM = 2  # untimed end-to-end calls first (page-locked buffers, host threads)

WORKLOADS = {
    "m100": dict(N=100_000, nus=[1.5], desc="Matern covariance N=100K full fp64 matrix, nu=1.5, "
                 "sigma2=1, beta=0.1, row-block sharded"),
    "m10": dict(N=10_000, nus=[1.5], desc="Matern covariance N=10K, nu=1.5, sigma2=1, beta=0.1"),
    "m50": dict(N=50_000, nus=[0.3, 0.8, 1.7, 2.9], desc="Matern covariance N=50K, nu sweep "
                "{0.3,0.8,1.7,2.9}, one matrix per nu per step"),
    "m200": dict(N=200_000, nus=[1.5], desc="Matern covariance N=200K lower-triangle tiles "
                 "(ts=256, packed, ~160 GB), area-balanced tile shards"),
    "bk": dict(n=64 << 20, desc="BesselK batch, 64Mi random (x,nu), x in (0,140], nu in (0,20]"),
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

    def init(self):
        import torch

        if torch.cuda.is_available():
            self.device_index = self.local % torch.cuda.device_count()
            torch.cuda.set_device(self.device_index)
        if self.world > 1 and self.pg is None:
            import torch.distributed as dist

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
# measured FP64 peak (roofline denominator)
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


# ---------------------------------------------------------------------------------------
# CPU reference (oracle port)
# ---------------------------------------------------------------------------------------

def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_matern_sample(N, nu, locs, target_s=12.0) -> dict:
    """Time the oracle's generate_covariance on a row-block sample, all host cores,
    and extrapolate to the compute-once full job: N(N+1)/2 computed entries."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    threads = cpu_threads()
    rows = 64
    t = 0.0
    while True:
        t0 = time.perf_counter()
        oracle.generate_covariance(locs, 1.0, 0.1, nu, row_range=(0, rows), threads=threads,
                                   tile_size=256)
        t = time.perf_counter() - t0
        if t >= target_s / 4 or rows >= N:
            break
        rows = min(N, int(rows * max(2.0, (target_s / 4) / max(t, 1e-3))))
    entries = rows * N
    rate = entries / t
    full = N * (N + 1) / 2 / rate
    return {"rate_entries_per_s": rate, "full_job_s": full, "threads": threads,
            "sample": f"rows [0,{rows}) x {N} cols of the nu={nu} matrix computed directly "
                      f"({entries:.3g} entries, {t:.2f} s) with oracle.generate_covariance "
                      f"on {threads} threads; extrapolated to the compute-once job "
                      f"N(N+1)/2 = {N * (N + 1) / 2:.4g} entries"}


def cpu_besselk_sample(x, nu, target_s=8.0) -> dict:
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    threads = cpu_threads()
    n = 1 << 18
    while True:
        t0 = time.perf_counter()
        oracle.refined_log_bessel_batch(x[:n], nu[:n], threads=threads)
        t = time.perf_counter() - t0
        if t >= target_s / 4 or n >= x.size:
            break
        n = min(x.size, int(n * max(2.0, (target_s / 4) / max(t, 1e-3))))
    return {"rate": n / t, "threads": threads, "n": n, "t": t}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------------
# workloads (ours)
# ---------------------------------------------------------------------------------------

def make_locs(N):
    return np.random.default_rng(SEED).random((N, 2))


def run_matern(args, D: Dist) -> dict:
    import torch

    import paper_2502_00356_b200 as bg
    from paper_2502_00356_b200 import _lib
    from paper_2502_00356_b200.covariance import _cov_launch, _lower_launch, matern_plan
    from paper_2502_00356_b200.distributed import computed_entries, row_shard, tile_shard

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
    pm = None
    mode = "rows"
    if packed:
        ntiles = bg.lower_tile_count(N, ts)
        l0, l1 = tile_shard(ntiles, D.world, D.rank)
        out = torch.empty((l1 - l0, ts, ts), dtype=torch.float64, device=dev)
        computed_local = float((l1 - l0) * ts * ts)  # diagonal tiles are stored complete
        stored_local = computed_local
    else:
        if D.world > 1 and args.mode in ("auto", "peer"):
            from paper_2502_00356_b200.distributed import MACRO, PeerMatrix

            try:
                pm = PeerMatrix(N, device=dev, mode=args.peer_layout)
                mode = "peer"
            except Exception as ex:  # noqa: BLE001 -- fall back to no-communication rows
                log(f"peer mapping unavailable ({ex}); using independent row blocks")
                if args.mode == "peer":
                    raise
        if pm is not None:
            r0, r1, out = pm.r0, pm.r1, pm.block
        if pm is not None and pm.mode == "band":
            from paper_2502_00356_b200.distributed import band_computed_entries

            computed_local = float(band_computed_entries(N, D.world, D.rank))
        elif pm is not None:
            lt = np.arange(*pm.tiles, dtype=np.int64)
            pp = ((np.sqrt(8.0 * lt + 1.0) - 1.0) // 2).astype(np.int64)
            pp += ((pp + 1) * (pp + 2) // 2 <= lt)
            pp -= (pp * (pp + 1) // 2 > lt)
            qq = lt - pp * (pp + 1) // 2
            mm = np.minimum(MACRO, N - MACRO * pp)
            nn_ = np.minimum(MACRO, N - MACRO * qq)
            computed_local = float(np.sum(mm * nn_))
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
           "computed_local": computed_local, "stored_local": stored_local, "N": N,
           "nus": nus, "mode": mode}
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
        theta = bg.MaternParams(1.0, 0.1, nus[0])
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        ts_ = []
        for k in range(E2E_WARM + e2e_steps):
            D.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for nu in nus:
                th = bg.MaternParams(1.0, 0.1, nu) if nu != nus[0] else theta
                bg.generate_covariance(locs, th, cfg, rows=(r0, r1), out=host)  # H2D locs, D2H rows
            torch.cuda.synchronize(dev)
            dt = time.perf_counter() - t0
            if k >= E2E_WARM:
                ts_.append(D.max(dt))
            else:
                D.max(dt)
        res["e2e_s"] = statistics.median(ts_)
        res["e2e_h2d"] = float(locs.nbytes) * D.world * len(nus)
        from paper_2502_00356_b200.covariance import host_d2h_bytes

        res["e2e_d2h"] = float(host_d2h_bytes(N, (r0, r1))) * len(nus)
        if r0 == 0 and r1 == N and res["e2e_d2h"] < stored * 8.0 * len(nus):
            from paper_2502_00356_b200.covariance import _host_threads

            res["e2e_how"] = (
                "paper_2502_00356_b200.generate_covariance(numpy locs, theta, out=pinned host "
                "array): H2D of the locations; per 1 GB row block the device computes the lower "
                f"part, a 2D copy moves it (half the matrix over PCIe) and {max(1, _host_threads() // 2)} host "
                "threads mirror it into the upper triangle (non-temporal stores) while the next "
                "block computes and copies; wall clock")
        del host
        release_host_cache()
    return res


def run_besselk(args, D: Dist) -> dict:
    import torch

    import paper_2502_00356_b200 as bg
    from paper_2502_00356_b200 import _lib
    from paper_2502_00356_b200.besselk import _launch_besselk

    n_total = WORKLOADS["bk"]["n"]
    dev = torch.device("cuda", D.device_index)
    from paper_2502_00356_b200.distributed import batch_shard

    i0, i1 = batch_shard(n_total, D.world, D.rank)
    rng = np.random.default_rng(SEED)
    x = 140.0 * (1.0 - rng.random(n_total))
    nu = 20.0 * (1.0 - rng.random(n_total))
    xd = torch.from_numpy(x[i0:i1]).to(dev)
    nd = torch.from_numpy(nu[i0:i1]).to(dev)
    stream = torch.cuda.current_stream(dev)
    cfg = bg.DEFAULT_CONFIG

    def step():
        return _launch_besselk(xd, nd, cfg, _lib.ROUTE_HYBRID, want_value=True, want_path=False)

    for _ in range(args.warmup):
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
    for _ in range(args.steps):
        step()
    e.record(stream)
    torch.cuda.synchronize(dev)
    launches = _lib.launch_count() - l0
    clk = clocks.stop() if D.rank == 0 else None
    ms = D.max(s.elapsed_time(e) / args.steps)
    res = {"ms_per_step": ms, "n": n_total, "launches": launches, "x": x, "nu": nu,
           "clocks": clk}
    # e2e: public API with host numpy arrays (H2D x, nu; D2H log K and K)
    if not args.no_e2e:
        tt = []
        # the host settles over the first few calls (page-locked allocations, then
        # ~40-80 ms calls, tools/bk_alloc_trace.py): more warm-up, median of 5
        warm = E2E_WARM + 2
        for k in range(warm + max(1, min(args.steps, args.e2e_steps + 2))):
            D.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            bg.bessel_k_batch(x[i0:i1], nu[i0:i1], cfg)  # the public API, validation included
            torch.cuda.synchronize(dev)
            dt = D.max(time.perf_counter() - t0)
            log(f"bk e2e call {k}: {dt * 1e3:.1f} ms")
            if k >= warm:
                tt.append(dt)
        res["e2e_s"] = statistics.median(tt)
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


def ncu_traffic(kernel: str, workload: str):
    """Per-unit DRAM traffic from the committed ncu --set full summary, if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            d = json.load(fh)
        return d.get(kernel, {}).get(workload)
    except (OSError, ValueError):
        return None


def ncu_pipe_frac(kernel: str):
    """The kernel's measured FP64-pipe utilisation (ncu, committed summary): the
    executed-op view of the roofline, next to the algorithmic-W `frac`."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            v = json.load(fh).get(kernel, {}).get("fp64_pipe_pct")
        return None if v is None else v / 100.0
    except (OSError, ValueError):
        return None


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
                    help="seconds of CPU work per reference / cpu_baseline sample")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to the contract minimum of 3")
        args.warmup = 3

    D = Dist()
    wl = WORKLOADS[args.workload]
    matern = args.workload != "bk"

    if args.impl == "reference":
        if D.rank != 0:
            return
        print(json.dumps(reference_line(args, D.world, wl, matern)), flush=True)
        return

    D.init()
    import torch

    peaks = peaks_file()
    fp64 = measure_fp64_peak(torch.device("cuda", D.device_index)) if D.rank == 0 else None

    # secondary: the BK batch line, single GPU only (keeps the default run short).  It
    # runs FIRST: after the M100 leg's 80 GB page-locked host buffer the host needs
    # seconds to settle, which would otherwise land in the BK end-to-end calls.
    sec = None
    if matern and not args.no_secondary and D.world == 1:
        a2 = argparse.Namespace(**vars(args))
        a2.steps, a2.warmup = 10, 3
        sec = run_besselk(a2, D)
        torch.cuda.empty_cache()

    if matern:
        r = run_matern(args, D)
    else:
        r = run_besselk(args, D)

    if D.rank == 0:
        line = build_line(args, D.world, wl, matern, r, sec, peaks, fp64)
        print(json.dumps(line), flush=True)
    D.barrier()
    D.close()


def build_line(args, world, wl, matern, r, sec, peaks, fp64):
    hbm = peaks.get("hbm_gbs", 6547.5)
    p64 = fp64["fp64_pipe_ops_per_s"]
    nominal = 148 * 64 * 1.965e9
    if matern:
        N = r["N"]
        nus = r["nus"]
        W = statistics.mean(W_MATERN.get(nu, 500.0) for nu in nus)
        t = r["ms_per_step"] * 1e-3
        # achieved over the timed region of rank 0's launches: computed entries per launch /
        # launch time (single launch per nu per step -> kernel time == step time / len(nus))
        kt = r["kernel_ms"] * 1e-3
        units_local = r["computed_local"]
        achieved = W * units_local / kt
        write_gbs = r["stored_local"] * 8.0 / kt / 1e9
        workload = args.workload
        metric = "Matern cov-gen time at N=100K" if workload == "m100" else \
            f"Matern cov-gen time ({wl['desc']})"
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
            "config": {"workload": f"{workload}: {wl['desc']}", "N": N, "nu": nus,
                       "sigma2": 1.0, "beta": 0.1, "bins": 40, "t_window": [0.0, 9.0],
                       "parallelism": (f"packed lower-tile shards x{world}" if workload == "m200" else
                                       f"fused compute + NVLink P2P mirror stores x{world}: each "
                                       f"64x64 tile pair computed once ({args.peer_layout} layout)"
                                       if r.get("mode") == "peer"
                                       else f"row-block shards x{world}, no collective"),
                       "l2": "output matrix (80 GB at N=100K) >> 126 MB L2; every step rewrites it"},
            "entries_per_s": r["stored_entries"] * len(nus) / t,
            "computed_entries_per_s": r["computed_entries"] * len(nus) / t,
            "roofline": {
                "bound": "fp64",
                "kernel": "bgk::matern_kernel",
                "achieved": achieved / 1e12,
                "peak": p64 / 1e12,
                "unit": "TFLOP/s",
                "op_convention": "FP64-pipe ops (DFMA = 1); W = 264 + 16*nbar = "
                                 f"{W:g} ops per computed entry (SURVEY.md 8d)",
                "frac": achieved / p64,
                "peak_source": fp64["how"] + f" (nominal 148x64x1.965GHz = {nominal / 1e12:.2f})",
                "traffic": ncu_traffic("matern_kernel", workload),
                "ncu_fp64_pipe_frac": ncu_pipe_frac("matern_kernel"),
                "hbm_write_gbs": write_gbs,
                "hbm_write_frac": write_gbs / hbm,
                "units_per_launch": units_local,
                "launch_ms": r["kernel_ms"],
            },
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
        }
        if "check_symmetric_diag_block" in r:
            line["check_symmetric_diag_block"] = r["check_symmetric_diag_block"]
        if "e2e_s" in r:
            line["e2e"] = {"value": r["e2e_s"], "unit": "s", "h2d_bytes_per_step": r["e2e_h2d"],
                           "d2h_bytes_per_step": r["e2e_d2h"],
                           "how": r.get("e2e_how",
                                        "paper_2502_00356_b200.generate_covariance(numpy locs, theta, "
                                        "rows=shard, out=pinned host array): H2D of the locations, "
                                        "device row blocks, D2H of every row (wall clock, max over ranks)")}
        if world == 1 and not args.no_cpu_baseline:
            locs = make_locs(N)
            c = cpu_matern_sample(N, nus[0], locs, target_s=args.cpu_sample_s)
            line["cpu_baseline"] = {"value": c["full_job_s"] * len(nus), "unit": "s",
                                    "cores": c["threads"], "kind": "port",
                                    "sample": c["sample"], "cpu": cpu_model()}
    else:
        n = r["n"]
        t = r["ms_per_step"] * 1e-3
        achieved = W_BESSELK * (n / world) / t
        line = {
            "metric": "BesselK evals/s", "value": n / t, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: x=140(1-U), nu=20(1-V), rng(20250201)",
            "config": {"workload": "bk: " + wl["desc"], "n": n,
                       "l2": "inputs+outputs 1.5 GB >> L2"},
            "roofline": {"bound": "fp64", "kernel": "bgk::besselk_kernel",
                         "achieved": achieved / 1e12, "peak": p64 / 1e12, "unit": "TFLOP/s",
                         "op_convention": "FP64-pipe ops, W = 700 per eval (SURVEY.md 8d)",
                         "frac": achieved / p64, "peak_source": fp64["how"],
                         "traffic": ncu_traffic("besselk_kernel", "bk"),
                         "ncu_fp64_pipe_frac": ncu_pipe_frac("besselk_kernel")},
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
        }
        if "e2e_s" in r:
            line["e2e"] = {"value": n / r["e2e_s"], "unit": "evals/s",
                           "h2d_bytes_per_step": 16.0 * n, "d2h_bytes_per_step": 17.0 * n}
        if world == 1 and not args.no_cpu_baseline:
            c = cpu_besselk_sample(r["x"], r["nu"], target_s=args.cpu_sample_s * 2 / 3)
            line["cpu_baseline"] = {"value": c["rate"], "unit": "evals/s", "cores": c["threads"],
                                    "kind": "port", "sample": f"first {c['n']} elements, "
                                    f"{c['t']:.2f} s", "cpu": cpu_model()}
    if sec is not None:
        t2 = sec["ms_per_step"] * 1e-3
        n2 = sec["n"]
        a2 = W_BESSELK * n2 / t2
        line["secondary"] = {
            "metric": "BesselK evals/s", "value": n2 / t2, "unit": "evals/s",
            "config": WORKLOADS["bk"]["desc"], "ms_per_step": sec["ms_per_step"],
            "roofline": {"kernel": "bgk::besselk_kernel", "achieved": a2 / 1e12,
                         "peak": p64 / 1e12, "unit": "TFLOP/s", "frac": a2 / p64,
                         "op_convention": "W = 700 FP64-pipe ops per eval (SURVEY.md 8d)",
                         "traffic": ncu_traffic("besselk_kernel", "bk"),
                         "ncu_fp64_pipe_frac": ncu_pipe_frac("besselk_kernel")},
        }
        if "e2e_s" in sec:
            line["secondary"]["e2e"] = {"value": n2 / sec["e2e_s"], "unit": "evals/s",
                                        "h2d_bytes_per_step": 16.0 * n2,
                                        "d2h_bytes_per_step": 17.0 * n2}
        if not args.no_cpu_baseline:
            c = cpu_besselk_sample(sec["x"], sec["nu"], target_s=args.cpu_sample_s * 2 / 3)
            line["secondary"]["cpu_baseline"] = {
                "value": c["rate"], "unit": "evals/s", "cores": c["threads"], "kind": "port",
                "sample": f"first {c['n']} elements of the same batch, {c['t']:.2f} s"}
    line["fp64_peak_measured_tops"] = p64 / 1e12
    return line


def reference_line(args, world, wl, matern) -> dict:
    """The reference's CPU algorithm (oracle port, bitwise equal to the numba kernels)
    on all host cores, bounded sample per step, same metric/unit/config."""
    if matern:
        N = wl["N"]
        nus = wl["nus"]
        locs = make_locs(N)
        per_step = []
        last = None
        for k in range(args.warmup + args.steps):
            tot = 0.0
            for nu in nus:
                last = cpu_matern_sample(N, nu, locs, target_s=(args.cpu_sample_s / 2
                                                                 if k >= args.warmup else
                                                                 args.cpu_sample_s / 12))
                tot += last["full_job_s"]
            if k >= args.warmup:
                per_step.append(tot)
        v = statistics.median(per_step)
        return {"impl": "reference", "metric": "Matern cov-gen time at N=100K" if args.workload == "m100"
                else f"Matern cov-gen time ({wl['desc']})", "value": v, "unit": "s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: rng(20250201).random((N,2)) unit-square locations",
                "config": {"workload": f"{args.workload}: {wl['desc']}", "N": N, "nu": nus},
                "cpu_baseline": {"value": v, "unit": "s", "cores": last["threads"],
                                 "kind": "port", "sample": last["sample"], "cpu": cpu_model()},
                "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    n = wl["n"]
    rng = np.random.default_rng(SEED)
    x = 140.0 * (1.0 - rng.random(n))
    nu = 20.0 * (1.0 - rng.random(n))
    rates = []
    last = None
    for k in range(args.warmup + args.steps):
        last = cpu_besselk_sample(x, nu, target_s=args.cpu_sample_s / 3)
        if k >= args.warmup:
            rates.append(last["rate"])
    v = statistics.median(rates)
    return {"impl": "reference", "metric": "BesselK evals/s", "value": v, "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": n / v * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "bk: " + wl["desc"], "n": n},
            "cpu_baseline": {"value": v, "unit": "evals/s", "cores": last["threads"], "kind": "port",
                             "sample": f"first {last['n']} elements", "cpu": cpu_model()},
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


if __name__ == "__main__":
    main()
