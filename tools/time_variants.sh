#!/bin/bash
# Time config E (and D) with every library variant in build/exp (one GPU call).
cd "$(dirname "$0")/.."
for so in build/exp/libqb_*.so; do
  tag=$(basename $so .so); tag=${tag#libqb_}
  echo "== $tag $(QB_LIB_PATH=$PWD/$so timeout 300 python tools/quick_times.py ${CONFIGS:-E} 2>&1 | tr '\n' ' ')"
done
