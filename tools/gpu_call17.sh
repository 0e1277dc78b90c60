mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
VARIANTS="base" SPECS="q2 mixed;dsv2 mixed;q15 mixed" bash tools/gpu_ab.sh > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu.log | head; cat gpurun_out/ab.txt
