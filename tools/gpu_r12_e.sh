#!/bin/bash
# sweep of the patched-immediate pass's fused-pair count (build/exp variants), then ncu of two of them
cd "$(dirname "$0")/.."
for so in build/exp/libqb_h*.so; do
  tag=$(basename $so .so)
  echo "== $tag"; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm_compare.py E 40 5 2>&1 | tail -2
done
for tag in h12 h14; do
  QB_LIB_PATH=$PWD/build/exp/libqb_$tag.so timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_imm_$tag python tools/profile_case.py E 40 5 > gpurun_out/ncu_imm_$tag.log 2>&1; echo "ncu $tag rc $?"
done
