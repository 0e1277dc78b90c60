#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bitexact.py tests/test_gpu_moe.py -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_ab${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab${TAG}.log
tail -3 gpurun_out/pytest_ab${TAG}.log
VARIANTS="${VARIANTS:-base}" SPECS="${SPECS:-q2 mixed;dsv2 mixed;q15 mixed;mx mixed;q2 w4a4_g128_sym}" bash tools/gpu_ab.sh
