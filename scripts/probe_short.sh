#!/bin/bash
# one-line-per-config summary of scripts/probe.py: build_s join merge finalize sample
python scripts/probe.py --no-warm "$@" 2>&1 | grep cfg | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); k=d['kernel_ms']; print(d['cfg'], d['build_s'], d['iters'], 'join', k['join'], 'merge', k['merge'], 'fin', k['finalize'], 'sample', k['sample'])
"
