#!/bin/bash
cd "$(dirname "$0")/.."
for so in build/exp/libqb_bm*.so; do echo "== $so"; QB_LIB_PATH=$PWD/$so timeout 120 python tools/batch_time.py; done
QB_LIB_PATH=$PWD/build/exp/libqb_bm0.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k batch 2>&1 | tail -1
