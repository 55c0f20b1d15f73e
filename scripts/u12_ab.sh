#!/bin/bash
O=gpurun_out/u12; mkdir -p $O
KNNG_JOIN_UTILES=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or step_matches or bit_exact" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/parity.log
tail -2 $O/parity.log
for cfg in C5; do
  KNNG_CUDA_LIB=scripts/libknng_cuda_head.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_head.json 2>&1
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_new.json 2>&1
  KNNG_CUDA_LIB=scripts/libknng_cuda_u12t192.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_t192.json 2>&1
  for v in head new t192; do python -c "
import json
for line in open('$O/probe_${cfg}_$v.json'):
    if line.startswith('{'):
        d=json.loads(line); print('$cfg', '$v', d['kernel_ms']['join'], [ (x[0], x[5]) for x in d['per_iter'][1:10]])
"; done
done
