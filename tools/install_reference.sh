#!/usr/bin/env bash
# Install the stock reference (pwadvect 0.1.0) into baseline/_ref, offline, for
# bench.py --impl reference and tests/test_gpu_reference_suite.py. Run in the
# dev container (needs /root/reference); baseline/_ref is git-ignored and
# travels to the GPU box with the gpurun snapshot. The reference's own tests
# and demos are copied beside the package, unmodified.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"          # the source tree is read-only; build from a copy
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
cp -r "$SRC/demos" "$ROOT/baseline/_ref/demos"   # the hot path's callers, run unchanged too
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
