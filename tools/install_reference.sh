#!/bin/sh
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot).  Used by
#   * bench.py --impl reference (times slbm.sparse.SparseEngine itself),
#   * tests/test_gpu_reference_suite.py (runs the reference's own test files
#     with the GPU engine swapped in, SURVEY §4 strategy 1),
#   * tests/test_gpu_integration.py (INTEGRATION.md §1 verbatim).
# The reference's tests are copied next to the install (baseline/_ref/
# slbm_tests) because /root/reference does not exist on the GPU box; nothing
# from the reference enters git history.
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/baseline/_ref" --upgrade "$TMP/pkg" >/dev/null
rm -rf "$HERE/baseline/_ref/slbm_tests"
cp -r "$SRC/tests" "$HERE/baseline/_ref/slbm_tests"
find "$HERE/baseline/_ref" -name __pycache__ -prune -exec rm -rf {} +
rm -rf "$TMP"
echo "reference installed in $HERE/baseline/_ref"
