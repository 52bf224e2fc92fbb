#!/bin/bash
# r13: IMM8 parity tests, then one ncu --set full capture of the threshold kernel at n=40
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests/test_gpu_imm.py -q -x --timeout 900 > gpurun_out/pytest_imm8.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_imm8.log
timeout 300 python tools/profile_case.py E 40 7 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:coarse8_kernel" -s 1 -c 1 -o gpurun_out/r13_ncu_imm8_E python tools/profile_case.py E 40 7 > gpurun_out/ncu_imm8.log 2>&1; echo "ncu rc $?"
