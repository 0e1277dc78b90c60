#!/bin/bash
# GPU parity suite (+ optional extra pytest args) -> gpurun_out/pytest_gpu.log
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
