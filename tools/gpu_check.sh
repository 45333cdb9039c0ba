#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, the ncu launch
# list of one fast pseudo-step and (optionally) an ncu --set full capture of
# the step's kernels.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_check.sh TAG [tests|notests] [full|nofull]
set -u
TAG=${1:-rx}
TESTS=${2:-tests}
FULL=${3:-full}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
if [ "$TESTS" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
  tail -3 $OUT/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench exit $?"; tail -c 3000 $OUT/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file $OUT/launches_$TAG.csv python tools/profile_step.py --steps 1 > $OUT/ncu_l_$TAG.log 2>&1
echo "ncu launches exit $?"
if [ "$FULL" = full ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o $OUT/full_$TAG python tools/profile_step.py --steps 1 > $OUT/ncu_f_$TAG.log 2>&1
  echo "ncu full exit $?"
fi
