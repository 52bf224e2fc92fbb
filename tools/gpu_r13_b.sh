#!/bin/bash
# r13: first run of the byte-packed threshold kernel (IMM8) against IMM, then the lazy-count variants
cd "$(dirname "$0")/.."
timeout 600 python tools/imm8_compare.py E 28,32,36,40 5 2>&1 | tee gpurun_out/imm8_first.log
timeout 300 python tools/imm8_compare.py D 32 5 2>&1 | tee -a gpurun_out/imm8_first.log
for so in build/exp/libqb_lazy*.so; do
  tag=$(basename $so .so); tag=${tag#libqb_}
  echo "== $tag"; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm8_compare.py E 40 5 2>&1 | grep imm8
done 2>&1 | tee gpurun_out/imm8_lazy.log
