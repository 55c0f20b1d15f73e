"""Where the host-pointer (e2e) build spends the time beyond the device build.

    python scripts/e2e_probe.py C2 [C5 ...]

Per config, five reps each: device-resident run_device; kg.run on pinned host
data (pageable numpy outputs, what bench.py's e2e times); the raw C-ABI with
pinned outputs; and the metrics' own split (iteration 0 = upload + byte check
+ init; the rest = iterations).
"""
import ctypes as C
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_06630_b200 as kg  # noqa: E402
from paper_2112_06630_b200 import _native as N, datasets  # noqa: E402
from paper_2112_06630_b200.knng import _metrics  # noqa: E402


def split(m):
    it0 = m.iterations[0].wall_time_s * 1e3
    rest = sum(it.wall_time_s for it in m.iterations[1:]) * 1e3
    return round(it0, 2), round(rest, 2), round(m.total_wall_time_s * 1e3, 2)


for name in sys.argv[1:] or ["C2"]:
    cfg = datasets.CONFIGS[name]
    data = datasets.generate(cfg)
    n, d = data.shape
    p = kg.RunParams(k=cfg.k, max_candidates=cfg.cap, seed=cfg.seed)
    dev = torch.from_numpy(data).cuda()
    ids = torch.empty((n, cfg.k), dtype=torch.int32, device="cuda")
    dists = torch.empty((n, cfg.k), dtype=torch.float32, device="cuda")
    pinned = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = data
    oid = torch.empty((n, cfg.k), dtype=torch.int32, pin_memory=True)
    odi = torch.empty((n, cfg.k), dtype=torch.float32, pin_memory=True)
    ofl = torch.empty((n, cfg.k), dtype=torch.uint8, pin_memory=True)
    import os
    out = {"cfg": name, "cpus": os.cpu_count(), "stage_kb": os.environ.get("KNNG_STAGE_KB")}

    def dev_run():
        m = kg.run_device(dev.data_ptr(), n, d, p, ids.data_ptr(), dists.data_ptr())
        torch.cuda.synchronize()
        return m

    def host_run():
        return kg.run(pinned.numpy(), p).metrics

    def raw_run():
        m, rows = _metrics(p.max_iterations + 1)
        cp = p._c()
        rc = N.lib().knng_cuda_run(pinned.data_ptr(), n, d, C.byref(cp), oid.data_ptr(),
                                   odi.data_ptr(), ofl.data_ptr(), None, C.byref(m))
        assert rc == 0
        return kg.RunMetrics._from_c(m, rows)

    def pageable_run():
        return kg.run(data, p).metrics

    for label, fn in (("device", dev_run), ("host_pageable_out", host_run),
                      ("host_pinned_out", raw_run), ("host_pageable_in_out", pageable_run)):
        fn()
        walls, splits = [], []
        for _ in range(5):
            t = time.perf_counter()
            m = fn()
            walls.append((time.perf_counter() - t) * 1e3)
            splits.append(split(m))
        out[label] = {"wall_ms": round(float(np.median(walls)), 2),
                      "it0_iters_total_ms": splits[len(splits) // 2]}
    print(json.dumps(out), flush=True)
