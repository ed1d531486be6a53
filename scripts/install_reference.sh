#!/bin/bash
# Install the UNMODIFIED reference package (bspb) into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun) and copy its test suite beside it, so that
# scripts/run_reference_suite.py can run the reference's own tests with the
# GPU batch drivers swapped in.  Needs /root/reference (this container only).
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree; the reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import bspb, bspb.kernels; print('bspb', bspb.__file__)"
