#!/bin/bash
# U tiles (join.cu tile_slab_u): parity with them on, then per-iteration join
# time with KNNG_JOIN_UTILES=0 / 1.
O=gpurun_out/ut; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py -x -q > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/parity.log
for cfg in ${CFGS:-C5 C4 C3 C1}; do
  for u in 0 1; do
    KNNG_JOIN_UTILES=$u timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_u$u.json 2>&1
  done
done
