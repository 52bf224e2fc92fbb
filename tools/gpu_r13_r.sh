#!/bin/bash
cd "$(dirname "$0")/.."
python tools/auto_zoo.py 38 2>&1 | tee gpurun_out/auto_zoo2.log
timeout 300 python tools/imm8_compare.py E 36,40 5 2>&1 | grep -E "imm8as|byte8" | awk '{print $2, $3, $5}'
timeout 1500 python -m pytest tests/test_gpu_imm.py -q -x --timeout 900 > gpurun_out/pytest_imm_r.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_imm_r.log
