#!/bin/bash
# one iteration: GPU tests, A/B timing of variants on each config, wait-site breakdown
mkdir -p gpurun_out; : > gpurun_out/ab.txt
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)" > gpurun_out/iter.txt
for c in ${CFGS:-dsv2 q15 q2 mx}; do CFG=$c STEPS=${STEPS:-10} bash tools/gpu_ab.sh > /dev/null 2>&1; done
for a in ${DIAG:-"dsv2 mixed"}; do timeout 300 python tools/diag_waits.py $a >> gpurun_out/iter.txt 2>&1; done
cat gpurun_out/iter.txt gpurun_out/ab.txt; grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head
