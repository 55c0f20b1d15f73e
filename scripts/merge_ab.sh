#!/bin/bash
O=gpurun_out/mrg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py -x -q -k "step_matches or hub or recall or determin" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/parity.log
tail -2 $O/parity.log
for cfg in C4 C5 C3 C2; do
  KNNG_CUDA_LIB=scripts/libknng_cuda_head.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_head.json 2>&1
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_new.json 2>&1
  for v in head new; do python -c "
import json
for line in open('$O/probe_${cfg}_$v.json'):
    if line.startswith('{'):
        d=json.loads(line); print('$cfg', '$v', d['build_s'], d['iters'], d['kernel_ms']['merge'])
    elif 'recall' in line: print(line.strip())
"; done
done
