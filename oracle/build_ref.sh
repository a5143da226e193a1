#!/bin/bash
# Installs the UNMODIFIED reference package (pure Python: /root/reference/pkg)
# into baseline/_ref for the two places that run the real reference:
#   * bench.py --impl reference (the CPU arm: rift2.match_pair on host cores)
#   * tests/test_ref_suite.py (the reference's own test modules, run against
#     this package through paper_2303_00319_b200.dropin.alias())
# The reference's test modules are copied next to the install
# (baseline/_ref/ref_tests).  baseline/_ref is git-ignored (never committed)
# but travels to the GPU box with the snapshot.  Test infrastructure only:
# nothing in the product package imports it.
set -eu
REF=${REF:-/root/reference/pkg}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
DEST="$ROOT/baseline/_ref"
[ -d "$REF/src/rift2" ] || { echo "reference not present at $REF: keeping $DEST as is"; exit 0; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"                      # the build writes egg-info next to the sources
rm -rf "$DEST"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DEST" "$TMP/pkg"
cp -r "$REF/tests" "$DEST/ref_tests"
echo "reference installed into $DEST"
