"""SASS instructions (with executed counts) attributed to given CUDA source lines.
usage: python tools/ncu_line_sass.py report.ncu-rep file.cu LINE [LINE...]"""
import csv
import io
import subprocess
import sys

rep, fname, lines = sys.argv[1], sys.argv[2], set(sys.argv[3:])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file = cur_line = None
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name"):
        continue
    if r[0]:
        cur_line = r[0]
        if cur_file == fname and cur_line in lines:
            print(f"--- {fname}:{cur_line} {r[1][:80]}")
        continue
    if cur_file == fname and cur_line in lines and r[2] not in ("...", "-"):
        print(f"   {r[7]:>12s} {r[4]:>6s}  {r[3].strip()[:70]}")
