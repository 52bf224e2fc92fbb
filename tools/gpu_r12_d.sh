#!/bin/bash
cd "$(dirname "$0")/.."
set -x
timeout 300 python tools/imm_compare.py E 40 5 > gpurun_out/imm_compare_E40.log 2>&1; echo "cmp rc $?"; cat gpurun_out/imm_compare_E40.log
timeout 300 python tools/imm_compare.py D 32 10 > gpurun_out/imm_compare_D32.log 2>&1; cat gpurun_out/imm_compare_D32.log
timeout 900 python -m pytest tests/test_gpu_imm.py -q -x > gpurun_out/pytest_imm.log 2>&1; echo "imm tests rc $?"; tail -15 gpurun_out/pytest_imm.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_imm_E python tools/profile_case.py E 40 5 \
    > gpurun_out/ncu_imm_E.log 2>&1; echo "ncu rc $?"
