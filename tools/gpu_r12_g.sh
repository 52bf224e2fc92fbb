#!/bin/bash
cd "$(dirname "$0")/.."
set -x
timeout 300 python tools/imm_compare.py E 40 5 2>&1 | tail -4
timeout 300 python tools/imm_compare.py D 32 10 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_imm.py -q > gpurun_out/pytest_imm2.log 2>&1; echo "imm tests rc $?"; grep -E "passed|failed|^FAILED" gpurun_out/pytest_imm2.log | tail
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse2_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_imm2_E python tools/profile_case.py E 40 6 > gpurun_out/ncu_imm2_E.log 2>&1; echo "ncu rc $?"
