"""Regenerate paper_2502_00356_b200/csrc/bgk_tables.cuh values (mpmath, 200 bits)."""
import mpmath

mpmath.mp.prec = 200
exp = [float(mpmath.power(2, mpmath.mpf(j) / 128)) for j in range(128)]
inv, lg = [], []
for j in range(128):
    c = 1 + (mpmath.mpf(j) + mpmath.mpf(0.5)) / 128
    ic = float(1 / c)
    inv.append(ic)
    lg.append(float(-mpmath.log(mpmath.mpf(ic))))
for name, vals in (("kExp2Tab128", exp), ("kInvC128", inv), ("kLogC128", lg)):
    print(name, ",".join(v.hex() for v in vals))
