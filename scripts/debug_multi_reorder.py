import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
cfg = datasets.CONFIGS["C1"]
data = datasets.generate(cfg)
reo = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=0, reorder=True, reorder_after_iteration=1)
for P in (1, 2):
    try:
        ids, dists, m = kg.run_multi(data, reo, num_gpus=P)
        print("P", P, "ok", len(m.iterations), flush=True)
    except Exception as e:
        print("P", P, "ERR", e, flush=True)
