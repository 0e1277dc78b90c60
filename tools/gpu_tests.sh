#!/bin/bash
# run the GPU test suites with hard timeouts; logs land in gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
for f in "$@"; do
  b=$(basename $f .py)
  timeout ${TEST_TIMEOUT:-600} python -m pytest $f -x -q -m gpu -p no:cacheprovider > gpurun_out/$b.log 2>&1
  echo "$f rc=$?" >> gpurun_out/summary.txt
  tail -15 gpurun_out/$b.log
done
