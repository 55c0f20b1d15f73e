#!/bin/bash
# A/B of the register-staged join (join_gl.cu) against the shared-memory tile
# kernel: parity with the path forced on, then per-iteration join time.
O=gpurun_out/gl; mkdir -p $O
KNNG_JOIN_GL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "step_matches or bit_exact or hub or recall_matches" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/parity.log
for cfg in ${CFGS:-C5 C3 C4}; do
  for gl in 0 1; do
    KNNG_JOIN_GL=$gl timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_gl$gl.json 2> $O/probe_${cfg}_gl$gl.err
  done
done
