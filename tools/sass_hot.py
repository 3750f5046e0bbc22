"""Code-size view of an ncu report: instructions executed at least once, and at least
`frac` x the max per-instruction count (the hot working set the i-cache must hold).
usage: python tools/sass_hot.py report.ncu-rep [frac]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[st:]))))
iE = rows[0].index("Instructions Executed")
cnt = []
for r in rows[1:]:
    try:
        cnt.append(int(r[iE]))
    except (ValueError, IndexError):
        pass
mx = max(cnt)
print(f"instructions {len(cnt)} ({16 * len(cnt) / 1024:.1f} KB), executed {sum(c > 0 for c in cnt)}, "
      f"hot(>= {frac} max) {sum(c >= frac * mx for c in cnt)} ({16 * sum(c >= frac * mx for c in cnt) / 1024:.1f} KB)")
