#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored; it
# travels to the GPU box with the repository snapshot) and copy its test
# suite next to it (baseline/_ref_tests, git-ignored) for the drop-in run
# (tests/test_dropin.py, dropin/sarfista).  Build from a scratch copy: the
# reference tree is read-only.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref" "$REPO/baseline/_ref_tests"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$REPO/baseline/_ref_tests"
rm -rf "$TMP"
echo "reference installed in $REPO/baseline/_ref, tests in $REPO/baseline/_ref_tests"
