#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python tools/auto_probe.py 2>&1 | tee gpurun_out/auto_probe.log
timeout 1500 python -m pytest tests/test_gpu_imm.py -q -x --timeout 900 > gpurun_out/pytest_imm8v.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_imm8v.log
