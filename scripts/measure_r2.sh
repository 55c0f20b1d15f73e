#!/bin/bash
# Round-2 measurement call (run under gpurun from the repo root).
set -x
O=gpurun_out/r2; mkdir -p $O
python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --sharded --config C4 --steps 2 --warmup 1 > $O/bench_sharded1_C4.json 2> $O/bench_sharded1_C4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_C5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:join_distances_kernel -s 0 -c 1 \
  -o $O/join_c5_iter1 -f python scripts/probe.py --no-warm --max-iter=1 C5 > $O/ncu_c5_1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:join_distances_kernel -s 7 -c 1 \
  -o $O/join_c5_iter8 -f python scripts/probe.py --no-warm --max-iter=8 C5 > $O/ncu_c5_8.log 2>&1
ls -la $O
