#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "E 32,36,40" "D 32,36,40" "B 40"; do set -- $cfg; timeout 600 python tools/imm8_compare.py $1 $2 3 2>&1 | grep -v "^Traceback" ; done | tee gpurun_out/imm8q.log
timeout 900 python tools/auto_probe.py 2>&1 | tee gpurun_out/auto_probe3.log
timeout 1500 python -m pytest tests/test_gpu_imm.py -q -x --timeout 900 > gpurun_out/pytest_imm8q.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_imm8q.log
