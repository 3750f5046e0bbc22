"""Per-CUDA-source-line stall samples and executed warp-instructions of an ncu report
(inlined code attributed to the line it came from).
usage: python tools/ncu_lines.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
stall = None  # optional: rank by one stall reason, e.g. NCU_STALL=stall_long_sb
import os
stall = os.environ.get("NCU_STALL")
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname = None
scol = 4
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        if stall and stall in r:
            scol = r.index(stall)
        break
res = []
tot_s = tot_i = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name"):
        continue
    if r[0] != "":
        try:
            s, n = int(r[scol]), int(r[7])
        except ValueError:
            continue
        res.append((s, n, f"{fname}:{r[0]}", r[1][:90]))
        tot_s += s
        tot_i += n
print(f"total samples {tot_s}, warp-inst {tot_i:.4g}")
for s, n, loc, src in sorted(res, reverse=True)[:topn]:
    print(f"{100 * s / tot_s:5.1f}% smp {100 * n / tot_i:5.1f}% inst  {loc:22s} {src}")

if len(sys.argv) > 3:  # phase ranges "name:lo-hi,..." over the main file's lines
    main = sys.argv[3].split("@")[0]
    ranges = [(p.split(":")[0], *map(int, p.split(":")[1].split("-"))) for p in sys.argv[3].split("@")[1].split(",")]
    agg = {}
    for s, n, loc, src in res:
        f, ln = loc.rsplit(":", 1)
        name = "other:" + f
        if f == main:
            for nm, lo, hi in ranges:
                if lo <= int(ln) <= hi:
                    name = nm
        a = agg.setdefault(name, [0, 0])
        a[0] += s
        a[1] += n
    for nm, (s, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{nm:40s} {100 * s / tot_s:5.1f}% samples {100 * n / tot_i:5.1f}% inst")
