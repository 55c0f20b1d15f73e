"""Joint (nn, no) histograms of the candidate lists at iterations 1, 3, 6 of a build
(GPU selection on the GPU build's graph state), saved as npz for tile models."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = datasets.CONFIGS[name]
data = datasets.generate(cfg)
out = {}
for it in (1, 2, 3, 4, 5, 6, 8, 10):
    res = kg.run(data, kg.RunParams(k=cfg.k, max_candidates=cfg.cap, max_iterations=it - 1)) if it > 1 else None
    if res is None:
        g, _, _ = kg.init_random(data, cfg.k, 1)
        ids, dists, flags = g.ids, g.dists, g.flags
    else:
        ids, dists, flags = res.graph.ids, res.graph.dists, res.graph.flags
    c, _ = kg.select_turbo(ids, dists, flags, cfg.cap, 7 + it)
    # joint histogram (nn, no), small enough to travel back
    h = np.zeros((cfg.cap + 1, cfg.cap + 1), np.int64)
    np.add.at(h, (c.new_counts.astype(np.int64), c.old_counts.astype(np.int64)), 1)
    out[f"h{it}"] = h
    print(name, it, "mean nn %.1f no %.1f" % (c.new_counts.mean(), c.old_counts.mean()), flush=True)
np.savez_compressed(f"gpurun_out/lists_{name}.npz", **out)
