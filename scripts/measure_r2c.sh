#!/bin/bash
# Round-2 final measurement call (run under gpurun from the repo root).
O=gpurun_out/r2c; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --impl reference > $O/bench_reference_C5.json 2> $O/bench_reference_C5.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
timeout 600 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_bench_C5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join5_kernel -s 7 -c 1 \
  -o $O/join5_c5_iter8 -f python scripts/probe.py --no-warm --max-iter=8 C5 > $O/ncu_c5_8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join5_kernel -s 5 -c 1 \
  -o $O/join5_c4_iter6 -f python scripts/probe.py --no-warm --max-iter=6 C4 > $O/ncu_c4_6.log 2>&1
head -c 600 $O/bench_C5.json; echo
ls -la $O
