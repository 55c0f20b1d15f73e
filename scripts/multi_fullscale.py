"""Full-scale parity of the in-process multi-GPU driver (knng_cuda_run_multi)
against the single-GPU build: same seed, recall@k on a 5000-node sample
against the exact K-NNG (GPU brute force).  On a one-GPU box all shards share
the device, so the times are not scaling numbers.

    python scripts/multi_fullscale.py C4 8
"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets

name = sys.argv[1]
shards = [int(x) for x in sys.argv[2:]] or [8]
cfg = datasets.CONFIGS[name]
data = datasets.generate(cfg)
params = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=cfg.seed)
q = np.random.default_rng(1).choice(cfg.n, size=min(cfg.n, 5000), replace=False).astype(np.uint32)
ex, _ = kg.brute_force_knng(data, cfg.k, queries=q)
t = time.time(); single = kg.run(data, params); ts = time.time() - t
out = {"config": name, "n": cfg.n, "single": {"recall": kg.recall(single.graph.ids[q], ex),
                                              "iterations": len(single.metrics.iterations) - 1,
                                              "wall_s": round(ts, 3)}}
for p in shards:
    t = time.time(); ids, dists, m = kg.run_multi(data, params, num_gpus=p); tm = time.time() - t
    out[f"shards_{p}"] = {"recall": kg.recall(ids[q], ex), "iterations": len(m.iterations) - 1,
                          "wall_s_one_gpu": round(tm, 3),
                          "evals": int(m.total_dist_evals)}
print(json.dumps(out), flush=True)
