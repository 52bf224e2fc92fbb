#!/bin/bash
cd "$(dirname "$0")/.."
for so in build/exp/libqb_k*.so; do
  tag=$(basename $so .so)
  echo "== $tag"; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm_compare.py E 40 5 2>&1 | grep imm2
done
QB_LIB_PATH=$PWD/build/exp/libqb_k10.so timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse2_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_imm2_k10 python tools/profile_case.py E 40 6 > gpurun_out/ncu_imm2_k10.log 2>&1; echo "ncu rc $?"
