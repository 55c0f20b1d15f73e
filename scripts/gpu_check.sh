#!/bin/bash
# GPU session: tests, per-iteration probes of C4/C5, ncu captures of the
# FP32 join on C4/C5 (iteration 1 and a late iteration).
O=gpurun_out/r2a; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python scripts/probe.py --no-warm C4 C5 > $O/probe_c4c5.log 2>&1
for c in C4 C5; do
  ncu --set full --clock-control none --import-source on -k regex:join_distances_kernel -s 0 -c 1 \
    -o $O/join_fp32_${c}_iter1 -f python scripts/probe.py --no-warm --max-iter=1 $c > $O/ncu_${c}_1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:join_distances_kernel -s 5 -c 1 \
    -o $O/join_fp32_${c}_iter6 -f python scripts/probe.py --no-warm --max-iter=6 $c > $O/ncu_${c}_6.log 2>&1
done
ls -la $O
