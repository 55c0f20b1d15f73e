#!/bin/bash
# Parity of a build variant (KNNG_CUDA_LIB) and probes of the default + variants.
O=gpurun_out/t5e; mkdir -p $O
KNNG_CUDA_LIB=scripts/libknng_cuda_$PVAR.so timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "variants or step_matches or bit_exact or distances" > $O/parity_$PVAR.log 2>&1; echo "pytest rc=$?" >> $O/parity_$PVAR.log
tail -3 $O/parity_$PVAR.log
for cfg in ${CFGS:-C5}; do
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_base.json 2>&1
  for v in ${VARS}; do
    KNNG_CUDA_LIB=scripts/libknng_cuda_$v.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_$v.json 2>&1
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/t5e/probe_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f.split("probe_")[1][:-5], "build_s", d["build_s"], "join", d["kernel_ms"]["join"], "iters", d["iters"],
                  [p[5] for p in d["per_iter"][1:10]])
PY
