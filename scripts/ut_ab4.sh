#!/bin/bash
O=gpurun_out/ut4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or step_matches or bit_exact" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/parity.log
tail -2 $O/parity.log
for cfg in ${CFGS:-C5}; do
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_new.json 2>&1
  KNNG_JOIN_UTILES=0 timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_u0.json 2>&1
done
for f in $O/probe_*.json; do echo $f; grep -o "\"join\": [0-9.]*" $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); print([ (x[0], x[5]) for x in d['per_iter'][1:10]])
"; done
