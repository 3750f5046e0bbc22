"""Print SASS lines (exec count + instruction) of an ncu report between two address suffixes.
usage: python tools/sass_range.py report.ncu-rep lo_hex hi_hex [lo hi ...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
rng = [(int(sys.argv[i], 16), int(sys.argv[i + 1], 16)) for i in range(2, len(sys.argv), 2)]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[st:]))))
h = rows[0]
iE, iS, iW = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
for r in rows[1:]:
    try:
        a = int(r[0], 16) & 0xfffff
    except ValueError:
        continue
    if any(lo <= a < hi for lo, hi in rng):
        print(f"{a:05x} {r[iE]:>10} {r[iW]:>6}  {r[iS]}")
