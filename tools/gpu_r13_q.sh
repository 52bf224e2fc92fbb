#!/bin/bash
cd "$(dirname "$0")/.."
for so in build/exp/libqb_*.so paper_2310_19373_b200/libqubrute_b200.so; do
  tag=$(basename $so .so); tag=${tag#libqb_}
  echo "== $tag"; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm8_compare.py E 32,36,38,40 5 2>&1 | grep -E "imm8as|byte8" | awk '{print $2, $3, $5}'
done 2>&1 | tee gpurun_out/imm8_cpt.log
