#!/bin/bash
# parity + NaN regression + A/B timing after a kernel change
mkdir -p gpurun_out; : > gpurun_out/check.txt
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)" >> gpurun_out/check.txt
for i in 1 2 3; do
  MXM_LIB=$(pwd)/tools/variants/lib_nan2.so NANTEST2=1 timeout 200 python tools/diag_mix.py 8 2048 14336 512 2 wa8,wo4 2>&1 | grep "nan rows" | sort | uniq -c >> gpurun_out/check.txt
done
for c in ${CFGS:-dsv2 q15 q2 mx}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /tmp/b.json 2>/tmp/b.err
  echo "$c rc=$? $(python -c 'import json; d=json.load(open("/tmp/b.json")); print("step_ms=%.4f gemm_ms=%.4f frac=%.3f" % (d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"]))' 2>&1 | tail -1)" >> gpurun_out/check.txt
done
cat gpurun_out/check.txt; grep -E "FAIL|Error|error" gpurun_out/pytest_gpu.log | head -20
