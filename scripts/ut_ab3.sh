#!/bin/bash
O=gpurun_out/ut3; mkdir -p $O
KNNG_JOIN_UTILES=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "step_matches or bit_exact or recall_matches" > $O/parity_u1.log 2>&1; echo "parity rc=$?" >> $O/parity_u1.log
for cfg in ${CFGS:-C4 C5 C3}; do
  KNNG_CUDA_LIB=scripts/libknng_cuda_head.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_head.json 2>&1
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_new.json 2>&1
done
tail -2 $O/parity_u1.log
for f in $O/probe_*.json; do echo $f; grep -o "\"join\": [0-9.]*" $f; done
