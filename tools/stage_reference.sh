#!/usr/bin/env bash
# Stage the UNMODIFIED reference (read-only /root/reference) into baseline/_ref so it travels to the
# GPU box with the gpurun snapshot (baseline/_ref is git-ignored, not gpurun-ignored):
#   * the package, installed offline exactly as the driver contract prescribes (pip --target);
#   * its own test suite (pkg/tests), which tests/test_reference_suite.py runs through both seams.
# Nothing here is committed; run it in the build container whenever /root/reference is present.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference}"
DST="$ROOT/baseline/_ref"
if [ ! -d "$SRC/pkg" ]; then echo "no reference at $SRC" >&2; exit 1; fi
TMP="$(mktemp -d)"
cp -r "$SRC/pkg" "$TMP/pkg"            # the build writes egg-info into the source tree: use a copy
rm -rf "$DST"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DST" "$TMP/pkg"
mkdir -p "$DST/qubrute_tests"
cp "$SRC"/pkg/tests/*.py "$DST/qubrute_tests/"
rm -rf "$TMP"
echo "staged reference package + $(ls "$DST/qubrute_tests" | wc -l) test files into $DST"
