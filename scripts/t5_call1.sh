#!/bin/bash
# Round-2 (session 6) call 1: full GPU suite with the 5x10 tile join as the
# default, probes per config, ncu of join5 on C5 / C4 iteration 1.
O=gpurun_out/t5; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
for cfg in C5 C4 C3 C1; do
  timeout 600 python scripts/probe.py $cfg > $O/probe_$cfg.json 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join5_kernel -s 0 -c 1 \
  -o $O/join5_c5_iter1 -f python scripts/probe.py --no-warm --max-iter=1 C5 > $O/ncu_c5_1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join5_kernel -s 2 -c 1 \
  -o $O/join5_c5_iter3 -f python scripts/probe.py --no-warm --max-iter=3 C5 > $O/ncu_c5_3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join5_kernel -s 0 -c 1 \
  -o $O/join5_c4_iter1 -f python scripts/probe.py --no-warm --max-iter=1 C4 > $O/ncu_c4_1.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/t5/probe_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(d["cfg"], "build_s", d["build_s"], d["kernel_ms"], "iters", d["iters"],
                  [p[5] for p in d["per_iter"][1:10]])
PY
ls -la $O
