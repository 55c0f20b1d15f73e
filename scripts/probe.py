"""Quick GPU probe: run kg.run on the configs with per-kernel profiling.

    python scripts/probe.py [--no-warm] [--max-iter N] C1 C2 ...
"""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets

args = [a for a in sys.argv[1:] if not a.startswith("--")]
warm = "--no-warm" not in sys.argv
max_iter = 30
for a in sys.argv[1:]:
    if a.startswith("--max-iter="):
        max_iter = int(a.split("=")[1])
names = args or ["C1", "C2", "C3"]
for name in names:
    cfg = datasets.CONFIGS[name]
    t = time.time(); data = datasets.generate(cfg); tg = time.time() - t
    p = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=cfg.seed, profile=True, max_iterations=max_iter,
                     reorder="--reorder" in sys.argv)
    if warm:
        kg.run(data[: min(len(data), 20000)], kg.RunParams(k=cfg.k, max_candidates=cfg.cap))
    t = time.time(); res = kg.run(data, p); wall = time.time() - t
    m = res.metrics
    print(json.dumps(dict(cfg=name, gen_s=round(tg, 2), wall_s=round(wall, 3), build_s=round(m.total_wall_time_s, 3),
        iters=len(m.iterations) - 1, evals=m.total_dist_evals, evals_per_s=m.total_dist_evals / m.total_wall_time_s,
        kernel_ms={k: round(v, 2) for k, v in m.kernel_ms.items()},
        per_iter=[(it.iteration, round(it.wall_time_s * 1e3, 2), it.dist_evals, it.changes, it.join_candidates, round(it.join_ms, 2)) for it in m.iterations])), flush=True)
    if cfg.n <= 200000 and max_iter >= 30:
        q = np.random.default_rng(1).choice(cfg.n, size=min(cfg.n, 5000), replace=False).astype(np.uint32)
        t = time.time(); ex, _ = kg.brute_force_knng(data, cfg.k, queries=q); tb = time.time() - t
        print(name, "recall(sample 5000)", kg.recall(res.graph.ids[q], ex), "bf_s", round(tb, 2), flush=True)
