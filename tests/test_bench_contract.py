"""bench.py's CPU-side contract: the reference arm (the reference's own CPU
implementation on the host cores -- its numba kernels from baseline/_ref when
installed, else the oracle port) prints exactly one JSON line with the contract's
keys, its K steps together run one whole job, and its config is the one our arm
prints; the N>1 mode selection falls back to row blocks when peer mapping fails."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_matern_line_is_one_whole_job():
    d = _run("--impl", "reference", "--workload", "m10", "--steps", "3", "--warmup", "3")
    assert d["impl"] == "reference" and d["unit"] == "s" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the K timed steps sum to the whole-job value, and the line fits its own run
    assert d["whole_job_measured"] and len(d["step_s"]) == 3
    assert abs(sum(d["step_s"]) - d["value"]) < 1e-9
    assert abs(d["ms_per_step"] * d["steps"] / 1e3 - d["value"]) < 1e-6
    assert d["check_symmetric"] is True
    import bench

    assert d["config"] == json.loads(json.dumps(bench.matern_config("m10", bench.WORKLOADS["m10"])))


def test_reference_arm_port_kind():
    d = _run("--impl", "reference", "--workload", "m10", "--steps", "1", "--warmup", "3",
             "--ref-kind", "port")
    assert d["cpu_baseline"]["kind"] == "port" and d["value"] > 0


def test_reference_arm_besselk_line():
    d = _run("--impl", "reference", "--workload", "bk1m", "--steps", "2", "--warmup", "3")
    assert d["metric"] == "BesselK evals/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["n"] == 1_000_000 and d["whole_job_measured"]


class _FakeDist:
    world, rank = 2, 0


def test_select_peer_falls_back_to_rows(monkeypatch):
    import argparse

    import bench
    import paper_2502_00356_b200.distributed as dist

    class Broken:
        def __init__(self, *a, **k):
            raise RuntimeError("cudaDeviceCanAccessPeer(0 -> 1) = 0")

    monkeypatch.setattr(dist, "PeerMatrix", Broken)
    args = argparse.Namespace(mode="auto", peer_layout="band")
    pm, mode, reason = bench.select_peer(args, _FakeDist(), 1000, None)
    assert pm is None and mode == "rows" and "CanAccessPeer" in reason
    args.mode = "peer"
    with pytest.raises(RuntimeError):
        bench.select_peer(args, _FakeDist(), 1000, None)
    args.mode = "rows"
    assert bench.select_peer(args, _FakeDist(), 1000, None) == (None, "rows", "--mode rows")
