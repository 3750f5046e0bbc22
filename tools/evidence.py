"""Summarise a tools/evidence.sh run (gpurun_out/*_TAG*) into profiles/:

  profiles/<TAG>_bench.json, <TAG>_reference.json   the two bench lines
  profiles/<TAG>_launches.csv                         ncu launch list (+ share table)
  profiles/<TAG>_ncu.json                             key metrics of the --set full captures
  profiles/ncu_summary.json                           what bench.py reads: per kernel the
      EXECUTED FP64-pipe ops per unit (sm__inst_executed_pipe_fp64.sum x 32 lanes / units),
      thread instructions per unit, issue-active and FP64-pipe %, full-size DRAM traffic,
      and the kernel-source hash of the build that was captured.

usage: python tools/evidence.py TAG
"""
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
sys.path.insert(0, R)
from bench import src_sha16  # noqa: E402

# units per captured launch (tools/profile_kernels.py): the N=20K full matrix computed
# once per entry pair (N(N+1)/2 entries, bench.py's convention) / 16Mi BK elements
UNITS = {"matern_kernel": 20000 * 20001 / 2, "besselk_kernel": float(1 << 24)}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, v = rows[0], rows[2]
    return {k: v[i] for i, k in enumerate(h)}


def num(d, k):
    try:
        return float(str(d[k]).replace(",", ""))
    except (KeyError, ValueError):
        return None


def rows(f):
    L = open(f).read().splitlines()
    i = next(k for k, l in enumerate(L) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(L[i:]))))


def traffic(f):
    d = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows(f)}
    return d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"], d


summary = {"_note": "bench.py roofline inputs, from tools/evidence.sh " + tag + " (ncu --set full "
           "captures: matern N=20K full matrix, besselk 16Mi BK elements; traffic: single-pass "
           "full-size launches)", "src_sha16": src_sha16()}
keys = {}
for kern, short, rep_key, traffic_key in (("matern_kernel", "matern", "m100", "m100"),
                                          ("besselk_kernel", "besselk", "bk", "bk")):
    rep = os.path.join(G, f"prof_{short}_{tag}.ncu-rep")
    if not os.path.exists(rep):
        continue
    d = raw(rep)
    u = UNITS[kern]
    fp64_warp = num(d, "sm__inst_executed_pipe_fp64.sum")
    warp = num(d, "smsp__inst_executed.sum")
    tpi = num(d, "smsp__thread_inst_executed_per_inst_executed.ratio")
    e = {"fp64_ops_per_unit": fp64_warp * 32 / u if fp64_warp else None,
         "thread_inst_per_unit": warp * tpi / u if warp and tpi else None,
         "warp_inst_per_unit_x32": warp * 32 / u if warp else None,
         "fp64_pipe_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
         "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
         "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
         "smem_bank_conflicts": num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
         "duration_ns": num(d, "gpu__time_duration.sum"),
         "sm_hz": num(d, "sm__cycles_elapsed.avg.per_second"),
         "registers": num(d, "launch__registers_per_thread"),
         "units": u, "src_sha16": summary["src_sha16"],
         "capture": f"gpurun_out/prof_{short}_{tag}.ncu-rep (profiles/{tag}_ncu.json)"}
    tf = os.path.join(G, f"traffic_{traffic_key}_{tag}.csv")
    if os.path.exists(tf):
        tot, det = traffic(tf)
        e["traffic"] = {rep_key: tot}
        e["traffic_detail"] = det
    summary[kern] = e
    keys[kern] = e
json.dump(summary, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
json.dump(keys, open(os.path.join(P, f"{tag}_ncu.json"), "w"), indent=1)
for src, dst in ((f"bench_{tag}.json", f"{tag}_bench.json"), (f"ref_{tag}.json", f"{tag}_reference.json"),
                 (f"launches_{tag}.csv", f"{tag}_launches.csv")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
lf = os.path.join(P, f"{tag}_launches.csv")
if os.path.exists(lf):
    t = defaultdict(float)
    n = defaultdict(int)
    for r in rows(lf):
        if r["Metric Name"] == "gpu__time_duration.sum":
            t[r["Kernel Name"][:48]] += float(r["Metric Value"].replace(",", ""))
            n[r["Kernel Name"][:48]] += 1
    tot = sum(t.values())
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        print(f"{100 * v / tot:5.1f}% {v / 1e6:9.3f} ms {n[k]:4d}x {k}")
print(json.dumps(keys, indent=1))
