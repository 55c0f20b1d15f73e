import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2112_06630_b200 as kg
O = oracle.load("restated")
def log(*a):
    print(*a, flush=True)
log("devices", kg.device_count())
data = np.random.default_rng(0).standard_normal((600, 24), dtype=np.float32)
t = time.time(); g, rev, ev = kg.init_random(data, 8, 5); log("init ok", time.time() - t, ev)
t = time.time(); c, fa = kg.select_turbo(g.ids, g.dists, g.flags, 15, 3); log("select ok", time.time() - t, c.new_counts.sum())
gi, cc, go, ch, ev = O.capture_step(data, 8, 15, 11, 1)
cands = kg.CandidateSet(cc.ids, cc.new_counts, cc.old_counts)
t = time.time(); D = kg.candidate_distances(data, cands); log("dist ok", time.time() - t, len(D))
t = time.time(); r = kg.compute_step(data, gi.ids, gi.dists, gi.flags, cands); log("join ok", time.time() - t, r[2], r[3], ch, ev)
t = time.time(); ids, dd = kg.brute_force_knng(data, 8); log("bf ok", time.time() - t)
t = time.time(); res = kg.run(data, kg.RunParams(k=8, max_candidates=15, profile=True)); log("run ok", time.time() - t, len(res.metrics.iterations))
log("recall", kg.recall(res.graph.ids, ids))
