"""Compare key metrics of ncu reports.  usage: python tools/ncu_cmp.py a.ncu-rep b.ncu-rep ..."""
import csv
import io
import subprocess
import sys

keys = [("gpu__time_duration.sum", "ms"), ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"), ("smsp__inst_executed.sum", "inst"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid")]
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    for r in rows[2:]:
        d = dict(zip(rows[0], r))
        out = [rep.split("/")[-1][:28], d.get("Kernel Name", "")[:30]]
        for k, n in keys:
            out.append(f"{n}={d.get(k, '?')}")
        st = {k[33:]: int(v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled")
              and not k.endswith("not_issued") and v.isdigit()}
        tot = sum(st.values()) or 1
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        print(" ".join(out))
        print("    stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
