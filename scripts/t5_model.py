"""FMA-pipe cost model of join5.cu's tiles on measured joint (nn, no)
histograms (scripts/list_sizes.py): units = packed FMA-pipe instructions per
8-float segment (fused tile 50, unfused 75).  Prints, per iteration, the live
share and the cost split by tile class, for the current tiling and variants."""
import sys
import numpy as np

def cur(nn, no, thinU=False, thinU2=False, pairF=False):
    fn, fo, m = nn - nn % 5, no - no % 5, nn + no
    nfb, nob = fn // 5, fo // 5
    blocks = sum(nfb - i + nob for i in range(nfb))
    f = sum((nfb - i + nob + 1) // 2 for i in range(nfb))
    if pairF: f = (blocks + 1) // 2
    r = nn - fn
    if r == 0: u = 0
    elif thinU and r <= 2: u = (m + 23) // 24
    else: u = (m + 9) // 10
    ro = no - fo
    if ro == 0 or fn == 0: u2 = 0
    elif thinU2 and ro <= 2: u2 = (fn + 23) // 24
    else: u2 = (fn + 9) // 10
    live_f = fn * (fn - 1) // 2 - nfb * 10 + nfb * 10 + fn * fo  # fused pairs (triangles included)
    live_u = nn * (nn - 1) // 2 + nn * no - live_f
    return 50 * f, 75 * u, 75 * u2, live_f, 1.5 * live_u

name = sys.argv[1]
z = np.load(f"gpurun_out/lists_{name}.npz")
for key in sorted(z.files, key=lambda s: int(s[1:])):
    h = z[key]
    tot = np.zeros(5)
    var = {"thinU": 0.0, "thinU+U2": 0.0, "pairF": 0.0, "all": 0.0}
    for nn, no in zip(*np.nonzero(h)):
        if nn == 0: continue
        w = h[nn, no]
        tot += w * np.array(cur(nn, no))
        var["thinU"] += w * sum(cur(nn, no, thinU=True)[:3])
        var["thinU+U2"] += w * sum(cur(nn, no, thinU=True, thinU2=True)[:3])
        var["pairF"] += w * sum(cur(nn, no, pairF=True)[:3])
        var["all"] += w * sum(cur(nn, no, True, True, True)[:3])
    cost = tot[:3].sum()
    print(f"{name} it {key[1:]:>2}: cost {cost:.3g} live {(tot[3] + tot[4]) / cost:.3f}  F {tot[0] / cost:.2f} U {tot[1] / cost:.2f} U2 {tot[2] / cost:.2f}"
          f"  liveF {tot[3] / max(tot[0], 1):.2f} liveU {tot[4] / max(tot[1] + tot[2], 1):.2f} | " +
          " ".join(f"{k} {v / cost:.3f}" for k, v in var.items()))

# --- merged leftover rows: new leftovers and old leftovers share row blocks ---
def merged(nn, no, thin):
    fn, fo, m = nn - nn % 5, no - no % 5, nn + no
    nfb, nob = fn // 5, fo // 5
    f = sum((nfb - i + nob + 1) // 2 for i in range(nfb))
    r, ro = nn - fn, (no - fo if fn else 0)
    def tiles(rows, cols):
        if rows == 0 or cols == 0: return 0
        if thin and rows <= 2: return (cols + 23) // 24
        return (cols + 9) // 10
    if r == 0: u = tiles(ro, fn)
    elif r + ro <= 5: u = tiles(r + ro, m) if not thin or r + ro > 2 else tiles(r + ro, m)
    else: u = tiles(r, m) + tiles(ro, fn)
    return 50 * f + 75 * u

print("merged leftover rows (plain / with 2x24 thin tiles), relative to current")
for key in sorted(z.files, key=lambda s: int(s[1:])):
    h = z[key]; base = a = b = 0.0
    for nn, no in zip(*np.nonzero(h)):
        if nn == 0: continue
        w = h[nn, no]
        base += w * sum(cur(nn, no)[:3]); a += w * merged(nn, no, False); b += w * merged(nn, no, True)
    print(f"{name} it {key[1:]:>2}: merged {a / base:.3f}  merged+thin {b / base:.3f}")

# --- the kept tiling (merged leftover rows; thin tiles for long rows): live share ---
print("kept tiling: live share of the FMA-pipe cost (thin tiles as for long rows / off)")
for key in sorted(z.files, key=lambda s: int(s[1:])):
    h = z[key]; a = b = live = 0.0
    for nn, no in zip(*np.nonzero(h)):
        if nn == 0: continue
        w = h[nn, no]
        c5 = cur(nn, no)
        live += w * (c5[3] + c5[4]); a += w * merged(nn, no, True); b += w * merged(nn, no, False)
    print(f"{name} it {key[1:]:>2}: live {live / a:.3f} / {live / b:.3f}")
