#!/bin/bash
# full GPU suite, bench line, launch list, ncu --set full of the default search kernel
cd "$(dirname "$0")/.."
set -x
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_j.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/pytest_gpu_j.log | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r12j.json 2> gpurun_out/bench_r12j.err; echo "bench rc $?"
tail -3 gpurun_out/bench_r12j.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_small_j.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r12_launches_j.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch_j.log 2>&1; echo "launch rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_imm_default python tools/profile_case.py E 40 0 > gpurun_out/ncu_imm_default.log 2>&1; echo "ncu rc $?"
