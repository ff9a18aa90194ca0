#!/bin/bash
# Run the reference's own test suite (pkg/tests, 224 tests) against the B200
# package through the package-swap shim (scripts/dropin/streambench).
#
#   here (no GPU; copies the reference tests into baseline/_ref/tests_ref, which
#   is git-ignored and travels to the GPU box with the snapshot):
#       bash scripts/run_reference_tests.sh --stage
#   on the GPU box:
#       bash scripts/run_reference_tests.sh [pytest args]
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
DEST="$ROOT/baseline/_ref/tests_ref"
if [ "${1:-}" = "--stage" ]; then
    mkdir -p "$DEST" && cp /root/reference/pkg/tests/*.py "$DEST/" && echo "staged $(ls "$DEST" | wc -l) files in $DEST"
    exit 0
fi
cd "$DEST" || { echo "no staged tests: run --stage in the build container first"; exit 2; }
PYTHONPATH="$ROOT/scripts/dropin:$ROOT" python -m pytest -q -p no:cacheprovider "$@" .
