#!/bin/bash
cd "$(dirname "$0")/.."
for so in build/exp/libqb_cw*.so; do echo "== $so"; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm_compare.py E 40 5 2>&1 | grep -E "imm "; QB_LIB_PATH=$PWD/$so timeout 300 python tools/imm_compare.py D 32 10 2>&1 | grep -E "imm "; done
QB_LIB_PATH=$PWD/build/exp/libqb_cw1.so timeout 900 python -m pytest tests/test_gpu_imm.py -q -x 2>&1 | tail -2
