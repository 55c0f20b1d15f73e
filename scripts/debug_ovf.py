"""Overflow -> grow -> rerun path vs the default buffer (deterministic mode)."""
import os, sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_2112_06630_b200 as kg
from test_gpu_parity import make_data

data = make_data("C1", 5000, 5)
p = kg.RunParams(k=20, max_candidates=20, seed=4, deterministic=True, profile=True)
for env in [{}, {"KNNG_TEST_DWORDS": "4096"}, {"KNNG_TEST_DWORDS": "4096", "KNNG_ITER_BATCH": "1"},
            {"KNNG_TEST_DWORDS": "200000"}]:
    for k in ("KNNG_TEST_DWORDS", "KNNG_ITER_BATCH"):
        os.environ.pop(k, None)
    os.environ.update(env)
    r = kg.run(data, p)
    print(env, [(it.iteration, it.dist_evals, it.changes, it.join_candidates) for it in r.metrics.iterations])
