#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r13t.json 2> gpurun_out/bench_r13t.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r13t.json 2> gpurun_out/bench_ref_r13t.err; echo "ref rc $?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_small_t.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r13_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch_t.log 2>&1; echo "launch rc $?"
head -c 400 gpurun_out/bench_r13t.json
