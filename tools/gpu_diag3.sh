#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/diag3.txt
run() { timeout 90 python tools/diag_mix.py "$@" > /tmp/o.txt 2>&1; echo "$* rc=$? $(grep -v CUDAEvent /tmp/o.txt | grep -m3 'ok\|Error' | tr '\n' ' ')" >> gpurun_out/diag3.txt; }
for i in 1 2 3; do run 8 2048 14336 512 2 wa8,wo4,wo4,wo4; done
for i in 1 2; do run 8 4096 14336 512 2 wa8,wo4,wo4,wo4; done
run 8 2048 14336 512 2 wa8,wo4
run 8 2048 14336 512 2 wa8
CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --config mx --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-comparators > /tmp/b.json 2>/tmp/b.err; echo "bench mx blocking rc=$? $(grep -v CUDAEvent /tmp/b.err | grep -B2 -m2 Error | tr '\n' ' ')" >> gpurun_out/diag3.txt
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/diag_mix.py 8 2048 14336 512 2 wa8,wo4,wo4,wo4 > gpurun_out/sanitizer.txt 2>&1; echo "sanitizer rc=$?" >> gpurun_out/diag3.txt
cat gpurun_out/diag3.txt; grep -v CUDAEvent gpurun_out/sanitizer.txt | head -60
