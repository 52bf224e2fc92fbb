#!/bin/bash
# final round-2 validation: full GPU suite, smoke, bench line, launch list
cd "$(dirname "$0")/.."
set -x
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_n.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR|SKIPPED" gpurun_out/pytest_gpu_n.log | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_n.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_n.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r12n.json 2> gpurun_out/bench_r12n.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r12n.json 2> gpurun_out/bench_ref_r12n.err; echo "ref rc $?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_small_n.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r12_launches_n.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch_n.log 2>&1; echo "launch rc $?"
