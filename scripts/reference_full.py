#!/usr/bin/env python
"""Full-config reference build (oracle/_ref: the unmodified knng headers), one
config per call, single-threaded as the reference is.  Writes
profiles/reference_full_<C>.json (per-iteration evals / changes / wall time,
build time, CPU model) and tests/golden/reference_rows_<C>.npz (the
reference's neighbour ids of bench.py's 5000-node recall sample, so the GPU
box can score the reference's recall against the same exact K-NNG as ours).

    python scripts/reference_full.py C5
"""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2112_06630_b200 import datasets  # noqa: E402


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    name = sys.argv[1]
    cfg = datasets.CONFIGS[name]
    t0 = time.time()
    data = datasets.generate(cfg)
    gen_s = time.time() - t0
    O = oracle.load("reference")
    r = O.run(data, k=cfg.k, cap=cfg.cap, delta=cfg.delta, seed=cfg.seed)
    n = cfg.n
    sample = np.random.default_rng(1).choice(n, size=min(n, 5000), replace=False).astype(np.uint32)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"reference_rows_{name}.npz"),
                        sample=sample, ids=r.graph.ids[sample].astype(np.uint32))
    out = {
        "config": name, "n": cfg.n, "d": cfg.d, "k": cfg.k, "cap": cfg.cap,
        "delta": cfg.delta, "seed": cfg.seed,
        "impl": "oracle/_ref (unmodified /root/reference/proj/include/knng, ref_harness.cpp)",
        "cpu": cpu_model(), "cores": 1,
        "iterations": r.iterations,
        "total_wall_s": r.total_wall,
        "total_evals": r.total_evals,
        "evals_per_s": r.total_evals / r.total_wall,
        "iter_evals": [int(x) for x in r.iter_evals],
        "iter_changes": [int(x) for x in r.iter_changes],
        "iter_wall_s": [float(x) for x in r.iter_wall],
        "datagen_s": gen_s,
    }
    with open(os.path.join(ROOT, "profiles", f"reference_full_{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if not k.startswith("iter_")}))


if __name__ == "__main__":
    main()
