mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head -20
VARIANTS="fat1 fat2 base" SPECS="mx mixed 1;mx mixed 16;mx mixed 64;mx mixed 512;dsv2 mixed;q15 mixed;q2 mixed" bash tools/gpu_ab.sh
