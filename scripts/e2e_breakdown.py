"""Where the host-pointer build's extra time goes (C2): H2D of the data alone,
D2H of the graph alone (pageable vs pinned), device-resident build, host build.

    python scripts/e2e_breakdown.py [C2]
"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = datasets.CONFIGS[name]
data = datasets.generate(cfg)
n, d = data.shape
pinned = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = data
dev = torch.empty((n, d), dtype=torch.float32, device="cuda")


def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print("h2d pinned ms", round(t(lambda: dev.copy_(pinned, non_blocking=True)), 3),
      "GB/s", round(n * d * 4 / t(lambda: dev.copy_(pinned, non_blocking=True)) / 1e6, 1))
g = torch.empty((n * cfg.k * 2,), dtype=torch.int32, device="cuda")
hp = np.empty(n * cfg.k * 2, np.int32)
hpin = torch.empty(n * cfg.k * 2, dtype=torch.int32, pin_memory=True)
print("d2h pageable ms", round(t(lambda: hp.__setitem__(slice(None), g.cpu().numpy())), 3))
print("d2h pinned ms", round(t(lambda: hpin.copy_(g, non_blocking=True)), 3))
p = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=cfg.seed)
ids = torch.empty((n, cfg.k), dtype=torch.int32, device="cuda")
dists = torch.empty((n, cfg.k), dtype=torch.float32, device="cuda")
dev.copy_(pinned)
print("device build ms", round(t(lambda: kg.run_device(dev.data_ptr(), n, d, p, ids.data_ptr(), dists.data_ptr())), 3))
host = pinned.numpy()
print("host build ms", round(t(lambda: kg.run(host, p)), 3))
