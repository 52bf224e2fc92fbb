#!/bin/bash
# round-2 call C: full GPU suite, issue-peak kernel, bench line
cd "$(dirname "$0")/.."
set -x
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_c.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/pytest_gpu_c.log
python tools/alu_peaks.py --out gpurun_out/r12_alu_peaks.json > gpurun_out/alu_peaks.log 2>&1; echo "alu rc $?"
grep issue gpurun_out/alu_peaks.log | cut -c1-300
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r12c.json 2> gpurun_out/bench_r12c.err; echo "bench rc $?"
cut -c1-3000 gpurun_out/bench_r12c.json
