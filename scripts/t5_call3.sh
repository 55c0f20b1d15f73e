#!/bin/bash
# Quick parity subset, probes (default + VARS), ncu of join5 on C4 iteration 1.
O=gpurun_out/t5c; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "variants or step_matches or bit_exact or distances" > $O/parity.log 2>&1; echo "pytest rc=$?" >> $O/parity.log
tail -3 $O/parity.log
for cfg in ${CFGS:-C5 C4 C3}; do
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_base.json 2>&1
  for v in ${VARS}; do
    KNNG_CUDA_LIB=scripts/libknng_cuda_$v.so timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_$v.json 2>&1
  done
done
for spec in ${NCU_SPECS}; do   # cfg:launches-to-skip
cfg=${spec%%:*}; skip=${spec##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join5_kernel -s $skip -c 1 \
  -o $O/join5_${cfg}_it$((skip+1)) -f python scripts/probe.py --no-warm --max-iter=$((skip+1)) $cfg > $O/ncu_${cfg}_$skip.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/t5c/probe_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f.split("probe_")[1][:-5], "build_s", d["build_s"], "join", d["kernel_ms"]["join"], "merge", d["kernel_ms"]["merge"], "iters", d["iters"],
                  [p[5] for p in d["per_iter"][1:10]])
PY
