#!/bin/bash
cd "$(dirname "$0")/.."
for so in build/exp/libqb_m5.so paper_2310_19373_b200/libqubrute_b200.so; do
  echo "== $so"; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm_compare.py E 40 5 2>&1 | grep -E "imm|coarse"
done
QB_LIB_PATH=$PWD/build/exp/libqb_m5.so timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_imm_m5 python tools/profile_case.py E 40 5 > gpurun_out/ncu_imm_m5.log 2>&1; echo "ncu rc $?"
