"""Pair-slot utilisation of tile layouts on measured (nn, no) list sizes."""
import sys
import numpy as np

def c(x, m): return (x + m - 1) // m * m

def tiles_cur(nn, no):
    fn, fo = nn - nn % 5, no - no % 5
    rows = list(range(fn)) + [None] * (c(fn, 8) - fn) + list(range(fn, nn)) + [None] * (c(nn - fn, 8) - (nn - fn))
    cf = list(range(fn)) + [nn + j for j in range(fo)]; cf += [None] * (c(len(cf), 8) - len(cf))
    cs = list(range(fn, nn)) + [nn + j for j in range(fo, no)]; cs += [None] * (c(len(cs), 8) - len(cs))
    return count(rows, cf + cs, nn, 8, 8)

def count(rows, cols, nn, R, C):
    slots = 0
    for r0 in range(0, len(rows), R):
        Rr = rows[r0:r0 + R]
        for c0 in range(0, len(cols), C):
            Cc = cols[c0:c0 + C]
            if any(i is not None and j is not None and (j >= nn or j > i) for i in Rr for j in Cc):
                slots += R * C
    return slots

def tiles_thin(nn, no):
    """fused rows x fused cols 8x8; remainder rows (<=4) as 4x16 tiles over all
    columns; fused rows x remainder cols as 16x4 tiles"""
    fn, fo = nn - nn % 5, no - no % 5
    rows_f = list(range(fn)) + [None] * (c(fn, 8) - fn)
    cf = list(range(fn)) + [nn + j for j in range(fo)]; cf += [None] * (c(len(cf), 8) - len(cf))
    rem_r = list(range(fn, nn)); rem_r += [None] * (c(len(rem_r), 4) - len(rem_r)) if rem_r else []
    cs = list(range(fn, nn)) + [nn + j for j in range(fo, no)]
    cs4 = cs + [None] * (c(len(cs), 4) - len(cs)) if cs else []
    allc = [x for x in cf if x is not None] + cs
    allc16 = allc + [None] * (c(len(allc), 16) - len(allc))
    s = count(rows_f, cf, nn, 8, 8)
    rf16 = rows_f + [None] * (c(len(rows_f), 16) - len(rows_f))
    if cs4: s += count(rf16, cs4, nn, 16, 4)
    if rem_r: s += count(rem_r, allc16, nn, 4, 16)
    return s

name = sys.argv[1]
z = np.load(f"gpurun_out/lists_{name}.npz")
for it in (1, 3, 6, 10):
    nn, no = z[f"nn{it}"], z[f"no{it}"]
    pairs = {}
    for a, b in zip(nn.tolist(), no.tolist()):
        if a: pairs[(a, b)] = pairs.get((a, b), 0) + 1
    U = sum(cnt * (a * (a - 1) // 2 + a * b) for (a, b), cnt in pairs.items())
    A = sum(cnt * tiles_cur(a, b) for (a, b), cnt in pairs.items())
    B = sum(cnt * tiles_thin(a, b) for (a, b), cnt in pairs.items())
    print(name, it, "useful %.3g" % U, "util current %.3f thin %.3f" % (U / A, U / B), "slots ratio %.3f" % (B / A))
