#!/bin/bash
# Run the reference's own unit tests against the B200 package (see sketchqr_alias.py).
#   here (container with /root/reference):  bash scripts/ref_suite/run.sh stage
#   GPU box:                                bash scripts/ref_suite/run.sh [patched] [test files...]
set -u
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
DST="$ROOT/baseline/_ref_tests"
if [ "${1:-}" = "stage" ]; then
  mkdir -p "$DST"
  cp /root/reference/pkg/tests/*.py "$DST"/
  ls "$DST"
  exit 0
fi
PLUGIN=sketchqr_alias
if [ "${1:-}" = "patched" ]; then  # the reference package itself, hot path through the C ABI (sketchqr_patch.py)
  PLUGIN=sketchqr_patch
  shift
fi
FILES=${@:-test_sketching.py test_rhqr.py test_linalg.py test_krylov.py test_trim.py test_experiments.py test_acceptance.py test_baselines.py}
cd "$DST" || { echo "stage the tests first (bash scripts/ref_suite/run.sh stage)"; exit 2; }
PYTHONPATH="$ROOT:$ROOT/scripts/ref_suite:$DST" python -m pytest -p $PLUGIN -p no:cacheprovider -q -rs \
  --tb=short --maxfail=400 $FILES
