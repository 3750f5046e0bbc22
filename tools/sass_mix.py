"""Summarise an ncu report's SASS page: executed warp-instructions by opcode and the
hottest instructions.  usage: python tools/sass_mix.py report.ncu-rep [kernel-regex]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
iS, iE, iT, iSamp = h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
mix = Counter()
samp = Counter()
tot = 0
hot = []
for r in rows[1:]:
    if len(r) <= iE:
        continue
    try:
        n = int(r[iE])
        s = int(r[iSamp])
    except ValueError:
        continue
    op = r[iS].strip().split()[0] if r[iS].strip() else "?"
    if op.startswith("@"):
        op = r[iS].strip().split()[1]
    base = op.split(".")[0]
    mix[base] += n
    samp[base] += s
    tot += n
    hot.append((s, n, r[0], r[iS].strip()))
print(f"total warp instructions: {tot:.4g}")
for op, n in mix.most_common(40):
    print(f"{op:10s} {n:14d} {100.0 * n / tot:6.2f}%  stall-samples {samp[op]}")
print("--- hottest by samples")
for s, n, a, src in sorted(hot, reverse=True)[:40]:
    print(f"{s:8d} {n:12d} {a[-5:]} {src}")
