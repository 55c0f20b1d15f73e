#!/bin/bash
# A/B of join_tc variants on C5 iterations 1-3 (join ms per iteration)
for v in "$@"; do
  lib=scripts/libknng_cuda_$v.so; [ "$v" = base ] && lib=paper_2112_06630_b200/lib/libknng_cuda.so
  echo "== $v"
  KNNG_CUDA_LIB=$lib KNNG_TC_STATS=1 timeout 300 python scripts/probe.py --max-iter=3 ${CFGS:-C5} 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['cfg'], [(it[0], it[5]) for it in d['per_iter']])
    elif 'prof' in l or 'Error' in l: print(l.strip())
"
done
