#!/bin/sh
# Run reference test files (from the read-only reference tree, never copied
# into this repo) against the B200 package through tools/refshim (htlr ->
# paper_2508_05958_b200).  Usage: tools/run_reference_tests.sh test_grids.py ...
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=/root/reference/pkg/tests
cd "$ROOT" || exit 1
args=""
for t in "$@"; do args="$args $REF/$t"; done
PYTHONPATH="$ROOT/tools/refshim:$ROOT:$REF" python -m pytest -q -p no:cacheprovider --rootdir "$ROOT/tools/refshim" $args
