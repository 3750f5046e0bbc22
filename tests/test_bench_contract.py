"""bench.py --impl reference runs on CPU (the reference arm: the oracle port on the
host cores) and prints exactly one JSON line with the contract's keys."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_matern_line():
    d = _run("--impl", "reference", "--workload", "m10", "--steps", "1", "--warmup", "3",
             "--cpu-sample-s", "0.4")
    assert d["impl"] == "reference" and d["unit"] == "s" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_besselk_line():
    d = _run("--impl", "reference", "--workload", "bk", "--steps", "1", "--warmup", "3",
             "--cpu-sample-s", "0.3")
    assert d["metric"] == "BesselK evals/s" and d["higher_is_better"] is True and d["value"] > 0
