#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "E 32,36,40" "D 36"; do set -- $cfg; timeout 600 python tools/imm8_compare.py $1 $2 3 2>&1 | grep -E "imm |imm8as|byte8|MATCH"; done | tee gpurun_out/byte8.log
timeout 900 python tools/auto_probe.py 2>&1 | tee gpurun_out/auto_probe4.log
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu_r13n.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|^FAILED|^ERROR|SKIPPED" gpurun_out/pytest_gpu_r13n.log | tail -15
