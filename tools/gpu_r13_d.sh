#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python tools/imm8_compare.py E 28,32,36,40 5 2>&1 | tee gpurun_out/imm8s_first.log
timeout 300 python tools/imm8_compare.py D 32 5 2>&1 | tee -a gpurun_out/imm8s_first.log
timeout 1500 python -m pytest tests/test_gpu_imm.py -q -x --timeout 900 > gpurun_out/pytest_imm8s.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_imm8s.log
