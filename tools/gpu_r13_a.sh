#!/bin/bash
# r13 baseline validation after the container was re-created: full GPU suite, smoke, both bench arms, launch list
cd "$(dirname "$0")/.."
set -x
nvidia-smi -L
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_r13a.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR|SKIPPED" gpurun_out/pytest_gpu_r13a.log | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r13a.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_r13a.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r13a.json 2> gpurun_out/bench_r13a.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r13a.json 2> gpurun_out/bench_ref_r13a.err; echo "ref rc $?"
which compute-sanitizer; timeout 300 compute-sanitizer --tool memcheck python tools/sanitize_case.py > gpurun_out/sanitize_r13a.log 2>&1; echo "sanitizer rc $?"; tail -5 gpurun_out/sanitize_r13a.log
cat gpurun_out/bench_r13a.json
