#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/diag_mix.txt
run() { timeout 60 python tools/diag_mix.py "$@" > /tmp/o.txt 2>&1; echo "$* rc=$? $(grep -v CUDAEvent /tmp/o.txt | grep -m3 'ok\|Error\|counts' | tr '\n' ' ')" >> gpurun_out/diag_mix.txt; }
run 8 4096 14336 512 2 wo4
run 8 2048 14336 512 2 wo4
run 2 256 14336 64 1 wo4
run 2 256 14336 64 1 wa8,wo4
run 8 2048 4096 512 2 wa8,wo4
run 8 2048 8192 512 2 wa8,wo4
run 8 2048 12288 512 2 wa8,wo4
run 8 2048 14336 512 2 wo2
run 8 2048 14336 512 2 w16
run 8 2048 14336 96 2 wo4
cat gpurun_out/diag_mix.txt
