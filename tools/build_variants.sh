#!/bin/bash
# Build experimental library variants into build/exp (each: tag + -D flags), in parallel.
cd "$(dirname "$0")/.."
mkdir -p build/exp
build_one() {
  tag=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -shared \
    "$@" -o build/exp/libqb_$tag.so paper_2310_19373_b200/csrc/qb_api.cu 2> build/exp/$tag.log && echo "built $tag"
}
while read -r tag flags; do
  [ -z "$tag" ] && continue
  build_one $tag $flags &
done
wait
