#!/bin/bash
# two-region H layout: GPU suite on the new build, workspace bytes and GEMM time vs the previous build (lib_old)
mkdir -p gpurun_out; O=gpurun_out/hsplit; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in q2 dsv2 q15; do
  timeout 300 python tools/ws_bytes.py $c >> $O/ws.txt 2>&1
  MXM_LIB=$(pwd)/tools/variants/lib_old.so timeout 300 python tools/ws_bytes.py $c >> $O/ws.txt 2>&1
done
NOTEST=1 VARIANTS="base old" SPECS="q2 mixed;dsv2 mixed;q15 mixed" TAG=16 bash tools/gpu_ab2.sh > /dev/null 2>&1
cp gpurun_out/ab16.txt $O/ 2>/dev/null
tail -3 $O/pytest_gpu.log; cat $O/ws.txt; cat $O/ab16.txt
