"""Minimax coefficients for the node exponential's polynomial (bgk_matern.cu kExpM).

p(r) = c0 + r (c1 + r (c2 + ... + r c_deg)) ~ e^r on |r| <= ln2 / 2^(bits+1), minimising
the maximum RELATIVE error (Remez exchange in mpmath, 50 digits).  Also writes the
correctly rounded table 2^(j/512), j = 0..511 (bgk_tables.cuh kExp2Tab512) with --table.
usage: python tools/remez_exp.py BITS DEG  |  python tools/remez_exp.py --table"""
import sys

import mpmath as mp

mp.mp.dps = 50


def remez(bits, deg):
    a = mp.log(2) / 2 ** (bits + 1)
    nc = deg + 1  # c0..c_deg
    n = nc + 1

    def err(c, r):
        q = sum(c[i] * r ** i for i in range(nc))
        return (q - mp.e ** r) / mp.e ** r

    pts = [a * mp.cos(mp.pi * (n - 1 - i) / (n - 1)) for i in range(n)]
    for _ in range(25):
        A, b = [], []
        for i, r in enumerate(pts):
            A.append([r ** j for j in range(nc)] + [-(-1) ** i * mp.e ** r])
            b.append(mp.e ** r)
        sol = mp.lu_solve(mp.matrix(A), mp.matrix(b))
        c = [sol[j] for j in range(nc)]
        grid = [-a + 2 * a * k / 3000 for k in range(3001)]
        ev = [err(c, r) for r in grid]
        ext = []
        for k in range(len(grid)):
            if k in (0, len(grid) - 1) or (abs(ev[k]) >= abs(ev[k - 1]) and abs(ev[k]) >= abs(ev[k + 1])):
                ext.append((grid[k], ev[k]))
        alt = []
        for r, e in ext:
            if alt and mp.sign(alt[-1][1]) == mp.sign(e):
                if abs(e) > abs(alt[-1][1]):
                    alt[-1] = (r, e)
            else:
                alt.append((r, e))
        while len(alt) > n:
            alt.pop(0 if abs(alt[0][1]) < abs(alt[-1][1]) else -1)
        pts = [r for r, e in alt]
    return c, max(abs(x) for x in ev)


if __name__ == "__main__":
    if sys.argv[1] == "--table":
        vals = [float(mp.mpf(2) ** (mp.mpf(j) / 512)).hex() for j in range(512)]
        for i in range(0, 512, 4):
            print("    " + ", ".join(vals[i:i + 4]) + ",")
    else:
        bits, deg = int(sys.argv[1]), int(sys.argv[2])
        c, e = remez(bits, deg)
        print(f"bits={bits} deg={deg} max rel err {mp.nstr(e, 4)}")
        print(", ".join(float(x).hex() for x in c))
