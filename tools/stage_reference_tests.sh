#!/bin/sh
# Stage the reference package and its own test files for the GPU box, where
# /root/reference does not exist (run in the build container). Both land in
# baseline/ (git-ignored, not gpurun-ignored), next to the pip install the
# reference arm uses; tests/test_gpu_reference_suite.py runs the staged tests
# against integration/octfield (the reference package with its hot path
# swapped for this repository's).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${REFERENCE_PKG:-/root/reference/pkg}
if [ ! -d "$ROOT/baseline/_ref/octfield" ]; then
  rm -rf /tmp/octfield_src && cp -r "$SRC" /tmp/octfield_src
  python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/octfield_src
fi
rm -rf "$ROOT/baseline/_ref_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref_tests"
echo "staged $(ls "$ROOT/baseline/_ref_tests" | wc -l) files in baseline/_ref_tests"
