#!/bin/bash
cd "$(dirname "$0")/.."
for so in build/exp/libqb_*.so; do
  tag=$(basename $so .so); tag=${tag#libqb_}
  echo "== $tag"; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm8_compare.py E 36,40 5 2>&1 | grep -E "imm8as|imm8a " | awk '{print $2, $3, $5}'
done 2>&1 | tee gpurun_out/imm8a_mb5.log
echo "== default"; timeout 300 python tools/imm8_compare.py E 36,40 5 2>&1 | grep -E "imm8as|imm8a " | awk '{print $2, $3, $5}'
