#!/bin/bash
# r15 validation of HEAD: GPU tests, smoke, bench (both arms), launch list
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_r15.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR|SKIPPED" gpurun_out/pytest_gpu_r15.log | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r15.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_r15.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r15.json 2> gpurun_out/bench_r15.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r15.json 2> gpurun_out/bench_ref_r15.err; echo "ref rc $?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_small_r15.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r15_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch_r15.log 2>&1; echo "launch rc $?"
head -c 600 gpurun_out/bench_r15.json
