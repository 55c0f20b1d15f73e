"""tcgen05 byte join vs the IMMA byte join on one fixed-state step (diagnostics)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
import oracle

O = oracle.load("restated")
data = datasets.generate(datasets.CONFIGS["C2"], 3000)
gi, c, go, _, ev_ref = O.capture_step(data, 20, 50, 1, int(sys.argv[1]) if len(sys.argv) > 1 else 1)
cands = kg.CandidateSet(c.ids, c.new_counts, c.old_counts)
os.environ["KNNG_U8_TC"] = "0"
g0 = kg.compute_step(data, gi.ids, gi.dists, gi.flags, cands)
print("imma done", flush=True)
os.environ["KNNG_U8_TC"] = "1"
g1 = kg.compute_step(data, gi.ids, gi.dists, gi.flags, cands)
print("tc done", flush=True)
same_ids = (g0[0].ids == g1[0].ids).mean()
same_d = (g0[0].dists.view(np.uint32) == g1[0].dists.view(np.uint32)).mean()
print("ids equal frac", same_ids, "dists equal frac", same_d, "evals", g0[3], g1[3], ev_ref, flush=True)
got0 = kg.candidate_distances(data, cands)
os.environ["KNNG_U8_TC"] = "0"
got1 = kg.candidate_distances(data, cands)
bad = sum(int((np.nan_to_num(got0[u]).view(np.uint32) != np.nan_to_num(got1[u]).view(np.uint32)).sum()) for u in got0)
print("candidate distance mismatches (tc vs imma):", bad, flush=True)
