#!/bin/bash
# Per-iteration join time of join.cu build variants (scripts/build_variants.py)
# on the configs in CFGS; default library first.
O=gpurun_out/var; mkdir -p $O
for cfg in ${CFGS:-C5 C3 C4}; do
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_base.json 2>&1
  for v in ${VARS}; do
    KNNG_CUDA_LIB=scripts/libknng_cuda_$v.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_$v.json 2>&1
  done
done
for cfg in ${STATCFGS}; do
  KNNG_CUDA_LIB=scripts/libknng_cuda_stats.so timeout 600 python scripts/join_stats.py $cfg > $O/stats_$cfg.txt 2>&1
done
