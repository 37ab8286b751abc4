#!/bin/bash
# Install the unmodified reference package into baseline/_ref (git-ignored; it
# travels to the GPU box with the gpurun snapshot) together with a copy of its
# own test suite, so the box can (1) time the real csemb CPU path next to the
# oracle port (bench.py --impl reference) and (2) run the reference's tests with
# the device seam installed (tests/test_reference_suite.py).  Needs
# /root/reference, i.e. runs in the build container only.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"   # the reference tree is read-only; setuptools writes build files
rm -rf "$ROOT/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
echo "reference installed into $ROOT/baseline/_ref (tests in baseline/_ref/tests)"
