"""In-degree distribution of a finished build (hubness check)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
for name in sys.argv[1:] or ["C2"]:
    cfg = datasets.CONFIGS[name]
    data = datasets.generate(cfg)
    res = kg.run(data, kg.RunParams(k=cfg.k, max_candidates=cfg.cap))
    deg = np.bincount(res.graph.ids.ravel().astype(np.int64), minlength=len(data))
    q = np.percentile(deg, [50, 90, 99, 99.9, 100])
    print(name, "in-degree p50/p90/p99/p99.9/max", q, "top5", np.sort(deg)[-5:], flush=True)
