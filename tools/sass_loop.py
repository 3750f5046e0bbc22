"""Print the hottest-looking FP64 loop body (a backward branch over >= 30 FP64 ops,
< 100 instructions) of one kernel in a cuobjdump -sass listing.
usage: cuobjdump -sass lib.so | python tools/sass_loop.py <kernel-substring>"""
import re
import sys

want = sys.argv[1]
cur, funcs = None, {}
for l in sys.stdin:
    m = re.search(r"Function : (\S+)", l)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
for name, ins in funcs.items():
    if want not in name:
        continue
    for a, t in ins:
        if "BRA" not in t:
            continue
        tg = re.search(r"0x([0-9a-f]+)", t)
        if not tg:
            continue
        ta = int(tg.group(1), 16)
        body = [x for x in ins if ta <= x[0] <= a]
        nfp = sum(1 for x in body if re.search(r"\bD(FMA|ADD|MUL)\b", x[1]))
        if ta < a and nfp >= int(sys.argv[2] if len(sys.argv) > 2 else 30) and len(body) < int(sys.argv[3] if len(sys.argv) > 3 else 100):
            print(f"{name}: loop {ta:#x}-{a:#x}, {len(body)} instructions, {nfp} FP64")
            for x in body:
                print(f"  {x[0]:#06x} {x[1]}")
            break
