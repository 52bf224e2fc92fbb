#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "E 32,36,40" "D 32,36,40" "B 32,40" "A 36"; do set -- $cfg; timeout 600 python tools/imm8_compare.py $1 $2 3 2>&1 | grep -v "^Traceback" ; done | tee gpurun_out/imm8_units.log
timeout 1500 python -m pytest tests/test_gpu_imm.py -q -x --timeout 900 > gpurun_out/pytest_imm8u.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_imm8u.log
