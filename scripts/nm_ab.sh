#!/bin/bash
# Tile order A/B (KNNG_JOIN_NODEMAJOR): parity with node-major on, then join ms.
O=gpurun_out/nm; mkdir -p $O
KNNG_JOIN_NODEMAJOR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or step_matches or bit_exact" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/parity.log
tail -2 $O/parity.log
for cfg in ${CFGS:-C5 C4 C3}; do
  for v in 0 1; do
    KNNG_JOIN_NODEMAJOR=$v timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_nm$v.json 2>&1
    echo $cfg nm$v $(grep -o "\"join\": [0-9.]*" $O/probe_${cfg}_nm$v.json)
  done
done
