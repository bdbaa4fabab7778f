#!/bin/bash
# Run the reference's own hot-path tests against the B200 drop-in (tools/refshim).
#
#   In the build container (reference present):  tools/refshim/run_reference_tests.sh stage
#       copies /root/reference/pkg/tests into baseline/_ref_tests (git-ignored scratch
#       that travels to the GPU box with baseline/_ref, the reference install).
#   On the GPU box:  tools/refshim/run_reference_tests.sh run [pytest args...]
#       writes gpurun_out/reftests.xml (junit, with each test's B200 entry points).
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
case "$1" in
  stage)
    rm -rf "$ROOT/baseline/_ref_tests"
    mkdir -p "$ROOT/baseline"
    cp -r /root/reference/pkg/tests "$ROOT/baseline/_ref_tests"
    rm -f "$ROOT"/baseline/_ref_tests/*.ts
    ;;
  run)
    shift
    cd "$ROOT/baseline/_ref_tests"
    mkdir -p "$ROOT/gpurun_out"
    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH="$ROOT/baseline/_ref:$ROOT:$ROOT/tools/refshim" \
      python -m pytest -p refshim_plugin -p no:cacheprovider -q -rfE \
      --junitxml="$ROOT/gpurun_out/reftests.xml" -o junit_family=xunit1 \
      . "$@"
    ;;
  *) echo "usage: $0 stage|run [pytest args]"; exit 2 ;;
esac
