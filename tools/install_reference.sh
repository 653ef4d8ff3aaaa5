#!/bin/bash
# Install the unmodified reference package (convkit 0.1.0) into baseline/_ref
# (git-ignored; it travels to the GPU box with the snapshot) and stage its
# test suite next to it for tests/test_gpu_reference_suite.py.  Nothing here
# is committed: the reference's sources never enter the repo's history.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=${1:-/root/reference}
[ -d "$REF/pkg" ] || { echo "no reference at $REF" >&2; exit 1; }
TMP=$(mktemp -d)
cp -r "$REF/pkg" "$TMP/pkg"   # the build writes into its source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$REF/pkg/tests" "$ROOT/baseline/_ref/convkit_tests"
rm -rf "$TMP"
echo "convkit installed in $ROOT/baseline/_ref"
