import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2112_06630_b200 as kg
import oracle
from test_gpu_parity import make_data
if not oracle.available("restated"):
    oracle.build("restated")
r = oracle.load("restated")
data = make_data("C3", 4000, 2)
gi, c, go, _, _ = r.capture_step(data, 30, 50, 2, 1)
g, rev, ch, ev = kg.compute_step(data, gi.ids, gi.dists, gi.flags, kg.CandidateSet(c.ids, c.new_counts, c.old_counts))
print("ok", ev)
