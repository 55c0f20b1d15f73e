"""Step-by-step run of one shard's phases with prints (diagnostics)."""
import sys, os
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200.shard import GpuShardEngine, seed_sequence

def p(*a):
    print(*a, flush=True)

data = np.random.default_rng(0).standard_normal((2000, 24)).astype(np.float32)
params = kg.RunParams(k=8, max_candidates=16, seed=3)
dd = torch.from_numpy(data).cuda()
p("create")
eng = GpuShardEngine(dd, params, 0, 1)
p("created", eng.lo, eng.hi, eng.seg_cap)
eng.init(1); torch.cuda.synchronize(); p("init")
ind = eng.degree(); torch.cuda.synchronize(); p("degree", int(ind.sum()))
counts, segs = eng.sample(2); p("sample", counts)
eng.offers(torch.empty(0, dtype=torch.int32, device="cuda")); torch.cuda.synchronize(); p("offers")
st = eng.step(); p("step", st["send_counts"], st["evals"], st["active"])
ch = eng.merge(torch.empty(0, dtype=torch.int32, device="cuda")); p("merge", ch)
ids, dists = eng.export(); torch.cuda.synchronize(); p("export", ids.shape)
eng.close(); p("closed")
for P in (2, 3):
    ids, dists, m = kg.run_multi(data, params, num_gpus=P); p("run_multi", P, len(m.iterations))
