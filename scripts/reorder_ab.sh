#!/bin/bash
# The locality reorder as a lever for the join (missing item 4):
# per-iteration join time with and without it, and ncu DRAM bytes / L2 hit rate
# of the join launch of iteration 4 (after the reorder at iteration 1).
O=gpurun_out/reorder; mkdir -p $O
for cfg in ${CFGS:-C4 C5}; do
  timeout 600 python scripts/probe.py $cfg > $O/probe_${cfg}_plain.json 2>&1
  timeout 600 python scripts/probe.py --reorder $cfg > $O/probe_${cfg}_reorder.json 2>&1
  for mode in plain reorder; do
    flag=""; [ $mode = reorder ] && flag="--reorder"
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_read.sum \
      --clock-control none -k regex:join5_kernel -s 3 -c 1 --csv --log-file $O/ncu_${cfg}_$mode.csv \
      python scripts/probe.py --no-warm --max-iter=4 $flag $cfg > $O/ncu_${cfg}_$mode.log 2>&1
  done
done
python - <<'PY'
import json,glob,csv
for f in sorted(glob.glob("gpurun_out/reorder/probe_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f.split("probe_")[1][:-5], "build_s", d["build_s"], "join", d["kernel_ms"]["join"], "reorder", d["kernel_ms"].get("reorder"), "merge", d["kernel_ms"]["merge"], "iters", d["iters"],
                  [p[5] for p in d["per_iter"][1:9]])
for f in sorted(glob.glob("gpurun_out/reorder/ncu_*.csv")):
    rows=[r for r in csv.reader(open(f)) if len(r)>5 and r[0].isdigit()]
    print(f.split("/")[-1], {r[-3]: r[-1]+" "+r[-2] for r in rows})
PY
