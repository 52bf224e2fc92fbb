#!/bin/bash
# Build experimental library variants into build/exp (stdin lines: "<tag> [-DFLAG=...]..."), one after
# another (each build already compiles its translation units in parallel).
cd "$(dirname "$0")/.."
mkdir -p build/exp
while read -r tag flags; do
  [ -z "$tag" ] && continue
  python -c "
import sys; sys.path.insert(0, '.')
from paper_2310_19373_b200 import _lib
_lib.build(output='build/exp/libqb_$tag.so', defines='$flags'.split())
" > build/exp/$tag.log 2>&1 && echo "built $tag" || echo "FAILED $tag (build/exp/$tag.log)"
done
