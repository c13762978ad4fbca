#!/bin/bash
# Install the unmodified reference (gmcf_mini, pure Python) into the
# git-ignored baseline/_ref -- the reference arm of bench.py and the CPU
# baseline time its own les.step / solve_pressure from there, on the GPU box
# too (baseline/_ref travels with the gpurun snapshot; /root/reference does
# not).  The reference's test suite is copied next to it (baseline/_ref/_tests)
# so tests/test_gpu_reference_suite.py can run it under install() on the box.
# Runs only where /root/reference exists (the build container).
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC; nothing to install"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"          # the reference tree is read-only; build from a copy
# numpy is already in the image; --no-deps skips the index-less resolution of it
python -m pip install -q --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/_tests"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref (tests in baseline/_ref/_tests)"
