#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "B 32,36,40" "D 36,40" "A 36"; do set -- $cfg; timeout 600 python tools/imm8_compare.py $1 $2 3 2>&1 | grep -v "^Traceback" ; done | tee gpurun_out/imm8_dense.log
