#!/bin/bash
cd "$(dirname "$0")/.."
set -x
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_f.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/pytest_gpu_f.log | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r12f.json 2> gpurun_out/bench_r12f.err; echo "bench rc $?"
cut -c1-2500 gpurun_out/bench_r12f.json
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_imm_final python tools/profile_case.py E 40 5 > gpurun_out/ncu_imm_final.log 2>&1; echo "ncu rc $?"
