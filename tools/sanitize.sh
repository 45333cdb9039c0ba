#!/bin/bash
# compute-sanitizer passes over the CUDA path on small grids:
# memcheck on smoke() + the scan-filter / scan-derivative / fused-stage GPU
# tests, racecheck and synccheck on smoke() and the scan kernels (cp.async
# rings and shared-memory scan carries).  Usage (GPU box, repo root):
#   bash tools/sanitize.sh TAG
# Writes gpurun_out/sanitize_<tool>_TAG.log; the last lines of each log carry
# the tool's "ERROR SUMMARY".
set -u
TAG=${1:-rx}
OUT=gpurun_out
mkdir -p $OUT
SMOKE='import __graft_entry__ as g; g.smoke()'
PYT_MEM="tests/test_gpu_filter_scan.py tests/test_gpu_deriv_scan.py::test_cylinder_curvature_c6_fast_vs_oracle tests/test_gpu_deriv_scan.py::test_annulus_hj_fast_vs_oracle tests/test_gpu_deriv_scan.py::test_annulus_256_full_segments tests/test_gpu_dist.py"
PYT_RACE="tests/test_gpu_filter_scan.py::test_scan_filter_vs_oracle tests/test_gpu_deriv_scan.py::test_annulus_hj_fast_vs_oracle"
run() {  # tool, label, timeout, command...
  local tool=$1 label=$2 tmo=$3
  shift 3
  local log=$OUT/sanitize_${tool}_${label}_$TAG.log
  timeout $tmo compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 "$@" > $log 2>&1
  local rc=$?
  echo "$tool/$label exit $rc: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)"
  echo "exit $rc" >> $log
}
run memcheck smoke 900 python -c "$SMOKE"
run memcheck tests 1500 python -m pytest -x -q -m gpu $PYT_MEM
run racecheck smoke 1200 python -c "$SMOKE"
run racecheck tests 1500 python -m pytest -x -q -m gpu $PYT_RACE
run synccheck smoke 900 python -c "$SMOKE"
run synccheck tests 1200 python -m pytest -x -q -m gpu $PYT_RACE
for f in $OUT/sanitize_*_$TAG.log; do echo "== $f"; tail -4 $f; done
