O=gpurun_out/r2b; mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
python bench.py --config C4 --steps 5 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_C5.json 2> $O/bench_ref_C5.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_C5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ls -la $O
