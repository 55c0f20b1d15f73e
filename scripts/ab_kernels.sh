#!/bin/bash
# A/B of library variants: per-category kernel ms of one build per config.
#   CFGS="C2 C3" scripts/ab_kernels.sh base d1 d3   (variant = scripts/libknng_cuda_<v>.so)
for v in "$@"; do
  lib=scripts/libknng_cuda_$v.so; [ "$v" = base ] && lib=paper_2112_06630_b200/lib/libknng_cuda.so
  KNNG_CUDA_LIB=$lib timeout 300 python scripts/probe.py ${CFGS:-C3} 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$v', d['cfg'], round(d['build_s'] * 1e3, 2), {k: v for k, v in d['kernel_ms'].items() if v})
"
done
