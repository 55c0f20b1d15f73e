#!/bin/bash
# Round-2 measurement after the bulk-staged init (run under gpurun).
set -x
O=gpurun_out/r2b; mkdir -p $O
python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
python bench.py --impl reference > $O/bench_reference_C5.json 2> $O/bench_reference_C5.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_C5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:join_distances_kernel -s 2 -c 1 \
  -o $O/join_c5_iter3 -f python scripts/probe.py --no-warm --max-iter=3 C5 > $O/ncu_c5_3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:init_random_bulk -s 0 -c 1 \
  -o $O/init_bulk_c5 -f python scripts/probe.py --no-warm --max-iter=1 C5 > $O/ncu_init.log 2>&1
ls -la $O
