#!/bin/bash
# A/B of the 5-aligned tile join (join5.cu) against the 8x8 tile kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "variants and T5" > gpurun_out/t5_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t5_test.log
tail -5 gpurun_out/t5_test.log
for cfg in ${T5_CFGS:-C5 C4 C3}; do
  for v in 0 1; do
    echo "== $cfg T5=$v" >> gpurun_out/t5_ab.log
    KNNG_JOIN_T5=$v timeout 600 python scripts/probe.py $cfg >> gpurun_out/t5_ab.log 2>&1
  done
done
python - <<'PY'
import json
for line in open("gpurun_out/t5_ab.log"):
    if line.startswith("=="): print(line.strip())
    elif line.startswith("{"):
        d = json.loads(line)
        print(d["cfg"], "build_s", d["build_s"], "join", d["kernel_ms"]["join"], "iters", d["iters"],
              [p[5] for p in d["per_iter"][1:9]])
PY
