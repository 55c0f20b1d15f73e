#!/bin/bash
# Timing-only experiment: iteration 1 of C5 with the per-slab CTA barrier
# replaced by a warp barrier (wrong results; bounds what removing the skew buys).
O=gpurun_out/t5d; mkdir -p $O
for v in base ${VARS}; do
  lib=paper_2112_06630_b200/lib/libknng_cuda.so; [ $v != base ] && lib=scripts/libknng_cuda_$v.so
  for mi in ${MAXIT:-1 3}; do
  KNNG_CUDA_LIB=$lib timeout 600 python scripts/probe.py --max-iter=$mi ${CFG:-C5} > $O/probe_${v}_$mi.json 2>&1
  python - <<PY
import json
for line in open("$O/probe_${v}_$mi.json"):
    if line.startswith("{"):
        d = json.loads(line); print("$v", "max-iter $mi", [p[5] for p in d["per_iter"][1:]], [p[2] for p in d["per_iter"][1:]])
PY
  done
done
