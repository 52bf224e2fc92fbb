#!/bin/bash
# r13 final validation
cd "$(dirname "$0")/.."
python tools/auto_zoo.py 38 2>&1 | tee gpurun_out/auto_zoo3.log
timeout 900 python tools/auto_probe.py 2>&1 | tee gpurun_out/auto_probe5.log
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_r13s.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR|SKIPPED" gpurun_out/pytest_gpu_r13s.log | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r13s.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_r13s.log
timeout 300 python tools/profile_case.py E 40 0 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:coarse8s_kernel" -s 1 -c 1 -o gpurun_out/r13_ncu_imm8as_final_E python tools/profile_case.py E 40 0 > gpurun_out/ncu_imm8as_final.log 2>&1; echo "ncu rc $?"
