#!/bin/bash
# r13 validation of the byte-packed kernels as AUTO's default: full GPU suite, smoke, ncu capture of the n=40
# search kernel (recorded for the bench's roofline), both bench arms, launch list
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_r13m.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR|SKIPPED" gpurun_out/pytest_gpu_r13m.log | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r13m.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_r13m.log
timeout 300 python tools/profile_case.py E 40 0 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:coarse8s_kernel" -s 1 -c 1 -o gpurun_out/r13_ncu_imm8as_plain_E python tools/profile_case.py E 40 0 > gpurun_out/ncu_imm8as_plain.log 2>&1; echo "ncu rc $?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r13m.json 2> gpurun_out/bench_r13m.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r13m.json 2> gpurun_out/bench_ref_r13m.err; echo "ref rc $?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_small_m.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r13_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch_m.log 2>&1; echo "launch rc $?"
head -c 600 gpurun_out/bench_r13m.json
