#!/bin/bash
O=gpurun_out/ut2; mkdir -p $O
for cfg in ${CFGS:-C4 C5 C3}; do
  KNNG_CUDA_LIB=scripts/libknng_cuda_head.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_head.json 2>&1
  for u in 0 1; do
    KNNG_JOIN_UTILES=$u timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_u$u.json 2>&1
  done
done
for f in $O/probe_*.json; do echo $f; grep -o "\"join\": [0-9.]*" $f; done
