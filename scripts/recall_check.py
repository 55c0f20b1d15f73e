"""GPU vs restated-reference recall@k on a config's generator at reduced n."""
import sys
sys.path.insert(0, ".")
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
import oracle
name = sys.argv[1]
cfg = datasets.CONFIGS[name]
if not oracle.available("restated"):
    oracle.build("restated")
r = oracle.load("restated")
for n in map(int, sys.argv[2:]):
    data = datasets.generate(cfg, n)
    ex, _ = kg.brute_force_knng(data, cfg.k)
    g = kg.run(data, kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=cfg.seed))
    ref = r.run(data, k=cfg.k, cap=cfg.cap, seed=cfg.seed)
    print(name, n, "gpu", round(kg.recall(g.graph.ids, ex), 4), "ref", round(kg.recall(ref.graph.ids, ex), 4),
          "iters", len(g.metrics.iterations) - 1, ref.iterations, flush=True)
