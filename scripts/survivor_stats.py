"""How many of the local join's pair evaluations can change the graph?

For iteration t's join state (captured from the CPU oracle) count, over all
evaluated pairs (a, b) of every node's new x new / new x old lists:

* ``kept``: pairs whose exact distance beats the iteration-start row maximum of
  a or b (the pairs the join writes as proposals today);
* ``pass_tf32``: pairs an approximate distance ||a||^2 + ||b||^2 - 2 a.b with
  a TF32 dot product cannot rule out (approx - bound < max(maxd[a], maxd[b]))
  with bound = 2 * 2^-10 * ||a|| ||b|| + fp32 slack;
* ``pass_3xtf32``: the same with a split (3-pass) TF32 dot product, bound
  2 * 2^-20 * ||a|| ||b||.

    python scripts/survivor_stats.py C2 20000 1 2 3 5 8
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2112_06630_b200 import datasets  # noqa: E402


def main():
    cfg = datasets.CONFIGS[sys.argv[1]]
    n = int(sys.argv[2])
    its = [int(x) for x in sys.argv[3:]] or [1, 2, 3]
    data = datasets.generate(cfg, n)
    O = oracle.load("restated")
    norms2 = (data.astype(np.float64) ** 2).sum(1)
    norms = np.sqrt(norms2)
    for t in its:
        gi, c, go, ch, ev = O.capture_step(data, cfg.k, cfg.cap, 0, t)
        maxd = gi.dists.max(1).astype(np.float64)
        cap = cfg.cap
        tot = kept = p1 = p3 = 0
        for u in range(n):
            nn, no = int(c.new_counts[u]), int(c.old_counts[u])
            if nn == 0:
                continue
            new = c.ids[u, :nn].astype(np.int64)
            old = c.ids[u, cap:cap + no].astype(np.int64)
            allr = np.concatenate([new, old])
            A = data[new].astype(np.float64)
            B = data[allr].astype(np.float64)
            dist = norms2[new][:, None] + norms2[allr][None, :] - 2 * A @ B.T
            mask = np.zeros((nn, nn + no), bool)
            iu = np.triu_indices(nn, 1)
            mask[iu] = True
            mask[:, nn:] = True
            thr = np.maximum(maxd[new][:, None], maxd[allr][None, :])
            nab = norms[new][:, None] * norms[allr][None, :]
            slack = 1e-6 * (norms2[new][:, None] + norms2[allr][None, :])
            tot += mask.sum()
            kept += (mask & (dist < thr)).sum()
            p1 += (mask & (dist - 2 * 2.0 ** -10 * nab - slack < thr)).sum()
            p3 += (mask & (dist - 2 * 2.0 ** -20 * nab - slack < thr)).sum()
        print(f"{cfg.name} n={n} t={t}: evals {tot} (ref {ev}) kept {kept / tot:.3f} "
              f"pass_tf32 {p1 / tot:.3f} pass_3xtf32 {p3 / tot:.3f}", flush=True)


if __name__ == "__main__":
    main()
