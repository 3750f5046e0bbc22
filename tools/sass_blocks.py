"""Per-basic-block executed-instruction share of an ncu report (SASS page).
usage: python tools/sass_blocks.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[st:]))))
h = rows[0]
iE, iS, iW = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
blocks, cur = [], None
for r in rows[1:]:
    try:
        n, w = int(r[iE]), int(r[iW])
    except ValueError:
        continue
    op = r[iS].split()
    op = (op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "")).split(".")[0]
    if cur and cur[1] == n:
        cur[2] += 1
        cur[3] += w
        cur[4].append(op)
    else:
        cur = [r[0][-5:], n, 1, w, [op]]
        blocks.append(cur)
tot = sum(b[1] * b[2] for b in blocks)
ws = sum(b[3] for b in blocks)
print(f"total warp-inst {tot:.4g}, stall samples {ws}")
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:topn]:
    c = Counter(b[4]).most_common(6)
    print(f"{b[0]} {b[1]:>10} x {b[2]:>4} = {100 * b[1] * b[2] / tot:5.1f}%  stall {100 * b[3] / ws:5.1f}%  {c}")
