"""List the loops (backward branches) of a kernel's SASS with instruction mix.
usage: python tools/sass_loops.py <lib.so> <mangled-kernel-name>"""
import re
import subprocess
import sys
from collections import Counter

txt = subprocess.run(["cuobjdump", "-sass", "-fun", sys.argv[2], sys.argv[1]],
                     capture_output=True, text=True).stdout
ins = []
for l in txt.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr = {a: i for i, (a, _) in enumerate(ins)}
FP = ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX")


def opc(t):
    t = t.strip()
    if t.startswith("@"):
        t = t.split(None, 1)[1]
    return t.split()[0].split(".")[0]


print("total instructions", len(ins))
for i, (a, t) in enumerate(ins):
    if "BRA" not in t:
        continue
    mm = re.findall(r"0x([0-9a-f]+)", t)
    if not mm:
        continue
    tgt = int(mm[-1], 16)
    if tgt < a and tgt in addr:
        body = ins[addr[tgt]:i + 1]
        c = Counter(opc(x[1]) for x in body)
        fp = sum(v for k, v in c.items() if k in FP)
        print(f"{tgt:#x} -> {a:#x} len {len(body)} fp64 {fp}", dict(c.most_common(9)))
