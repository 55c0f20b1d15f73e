#!/bin/bash
# One measurement call for profiles/ (run under gpurun from the repo root):
#   bench lines of C1-C5 and the reference arm, the C2 launch list, and ncu
#   --set full captures of the two join kernels' iteration-1 launches.
# Then, in the container: python scripts/make_profiles.py <tag>
set -x
O=gpurun_out/prof; mkdir -p $O
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for c in C1 C3 C4 C5; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
python bench.py --impl reference > $O/bench_reference_C2.json 2> $O/bench_reference_C2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_C2.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:join_u8_kernel -s 0 -c 1 \
  -o $O/join_u8_c2_iter1 -f python scripts/probe.py --no-warm --max-iter=1 C2 > $O/ncu_u8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:join_distances_kernel -s 0 -c 1 \
  -o $O/join_fp32_c3_iter1 -f python scripts/probe.py --no-warm --max-iter=1 C3 > $O/ncu_fp32.log 2>&1
ls -la $O
