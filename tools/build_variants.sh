#!/bin/bash
# Build experimental library variants: tools/build_variants.sh tag "-DFLAGS..." ...
cd "$(dirname "$0")/.."
build_one() {
  tag=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -shared \
    "$@" -o build/exp/libqb_$tag.so paper_2310_19373_b200/csrc/qb_api.cu 2> build/exp/$tag.log && echo "built $tag"
}
build_one base &
build_one mb5 -DQB_MINB=5 &
build_one mb6 -DQB_MINB=6 &
build_one b54 -DQB_BIG_B1=5 -DQB_BIG_B2=4 &
build_one b54mb6 -DQB_BIG_B1=5 -DQB_BIG_B2=4 -DQB_MINB=6 &
build_one b64 -DQB_BIG_B1=6 -DQB_BIG_B2=4 &
build_one tpb256mb2 -DQB_TPB=256 -DQB_MINB=2 &
build_one b45 -DQB_BIG_B1=4 -DQB_BIG_B2=5 -DQB_MINB=6 &
wait
