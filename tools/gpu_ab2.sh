#!/bin/bash
# GPU tests (product build) then A/B GEMM timing of library variants over configs
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_ab${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab${TAG}.log
tail -3 gpurun_out/pytest_ab${TAG}.log
fi
VARIANTS="${VARIANTS:-base}" SPECS="${SPECS:-q2 mixed;dsv2 mixed;q15 mixed;mx mixed;q2 w4a4_g128_sym;q2 w8a8_g-1_sym}" bash tools/gpu_ab.sh
