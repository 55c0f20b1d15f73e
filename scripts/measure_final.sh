#!/bin/bash
# Final round-2 check: full GPU suite, smoke(), bench lines on the final code.
O=gpurun_out/final; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --impl reference > $O/bench_reference_C5.json 2> $O/bench_reference_C5.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
python - <<'PY'
import json
for c in ["C5","C4","C3","reference_C5"]:
    try:
        d=json.loads(open(f"gpurun_out/final/bench_{c}.json").read().strip().splitlines()[-1])
        print(c, "value %.4g"%d["value"], "ms", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"), d.get("recall_at_k"))
    except Exception as e: print(c, "ERR", e)
PY
