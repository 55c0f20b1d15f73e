import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2112_06630_b200 as kg
from paper_2112_06630_b200 import datasets
cfg = datasets.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
data = datasets.generate(cfg); n, d = data.shape
dd = torch.from_numpy(data).cuda(); ids = torch.empty((n, cfg.k), dtype=torch.int32, device="cuda"); ds = torch.empty((n, cfg.k), device="cuda")
for prof in (False, True):
    p = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, profile=prof)
    for _ in range(2): kg.run_device(dd.data_ptr(), n, d, p, ids.data_ptr(), ds.data_ptr())
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): m = kg.run_device(dd.data_ptr(), n, d, p, ids.data_ptr(), ds.data_ptr())
    torch.cuda.synchronize(); print("device profile=%s %.1f ms" % (prof, (time.perf_counter() - t) * 200), m.total_wall_time_s * 1e3, flush=True)
    for _ in range(2): kg.run(data, p)
    t = time.perf_counter()
    for _ in range(5): r = kg.run(data, p)
    print("host   profile=%s %.1f ms" % (prof, (time.perf_counter() - t) * 200), r.metrics.total_wall_time_s * 1e3, flush=True)
