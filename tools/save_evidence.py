"""Copy a round_evidence.sh run (gpurun_out/*_TAG*) into profiles/: bench line, reference
arm, launch list, ncu key metrics, and the full-size traffic / pipe summary that
bench.py reads (profiles/ncu_summary.json).  usage: python tools/save_evidence.py TAG"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1]
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(R, "gpurun_out"), os.path.join(R, "profiles")


def rows(f):
    L = open(f).read().splitlines()
    i = next(k for k, l in enumerate(L) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(L[i:]))))


def rd(f):
    return {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows(f)}


reps = [os.path.join(G, f"prof_{k}_{tag}.ncu-rep") for k in ("matern", "besselk")]
out = subprocess.run([sys.executable, os.path.join(R, "tools", "ncu_summary.py"), *reps],
                     capture_output=True, text=True, check=True).stdout
open(os.path.join(P, f"r01_ncu_{tag}.json"), "w").write(out)
shutil.copy(os.path.join(G, f"bench_full_{tag}.json"), os.path.join(P, f"r01_bench_full_{tag}.json"))
shutil.copy(os.path.join(G, f"bench_ref_{tag}.json"), os.path.join(P, f"r01_bench_reference_{tag}.json"))
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, "r01_launches.csv"))
nv = json.loads(out)


def pct(k):
    for kk, v in nv.items():
        if k in kk:
            return float(v["fp64_pipe_pct"].split()[0])


m, b = rd(os.path.join(G, "traffic_m100.csv")), rd(os.path.join(G, "traffic_bk.csv"))
src = "ncu --set full, sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, {} (profiles/r01_ncu_%s.json)" % tag
s = {"_note": "per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) from single-pass "
              "ncu captures of the full-size launches on B200 (tools/profile_traffic.sh, round 1, "
              f"{tag} kernels); used by bench.py as roofline.traffic",
     "matern_kernel": {"m100": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"], "m100_detail": m,
                       "fp64_pipe_pct": pct("matern"),
                       "fp64_pipe_source": src.format("N=20K full-matrix launch")},
     "besselk_kernel": {"bk": b["dram__bytes_read.sum"] + b["dram__bytes_write.sum"], "bk_detail": b,
                        "fp64_pipe_pct": pct("besselk"),
                        "fp64_pipe_source": src.format("16Mi-element launch")}}
json.dump(s, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
t = defaultdict(float)
for r in rows(os.path.join(P, "r01_launches.csv")):
    if r["Metric Name"] == "gpu__time_duration.sum":
        t[r["Kernel Name"][:40]] += float(r["Metric Value"].replace(",", ""))
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda x: -x[1]):
    print(f"{100 * v / tot:5.1f}% {v / 1e6:9.3f} ms {k}")
for k, v in nv.items():
    print(k.split(":")[-1][:40], v["duration"], v["fp64_pipe_pct"], v["issue_active_pct"])
print("traffic m100", m, "bk", b)
