#!/bin/bash
O=gpurun_out/agg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py -x -q -k "variants or step_matches or bit_exact or hub or recall_matches or determin" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/parity.log
tail -2 $O/parity.log
for cfg in ${CFGS:-C5 C4 C3 C1}; do
  KNNG_CUDA_LIB=scripts/libknng_cuda_head.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_head.json 2>&1
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_new.json 2>&1
  echo $cfg head $(grep -o "\"join\": [0-9.]*" $O/probe_${cfg}_head.json) new $(grep -o "\"join\": [0-9.]*" $O/probe_${cfg}_new.json)
done
