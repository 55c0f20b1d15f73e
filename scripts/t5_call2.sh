#!/bin/bash
# Parity of the reworked join5 tiles, then per-config probes of the default
# library and the build variants in VARS.
O=gpurun_out/t5b; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -m gpu > $O/parity.log 2>&1; echo "pytest rc=$?" >> $O/parity.log
tail -4 $O/parity.log
for cfg in ${CFGS:-C5 C4 C3}; do
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_base.json 2>&1
  for v in ${VARS}; do
    KNNG_CUDA_LIB=scripts/libknng_cuda_$v.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_$v.json 2>&1
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/t5b/probe_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f.split("probe_")[1][:-5], "build_s", d["build_s"], "join", d["kernel_ms"]["join"], "merge", d["kernel_ms"]["merge"], "iters", d["iters"],
                  [p[5] for p in d["per_iter"][1:10]])
PY
