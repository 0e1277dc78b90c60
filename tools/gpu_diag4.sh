#!/bin/bash
mkdir -p gpurun_out
FILLTEST=1 timeout 200 python tools/diag_mix.py 8 2048 14336 512 2 wa8,wo4,wo4,wo4 > gpurun_out/diag4.txt 2>&1
grep -v CUDAEvent gpurun_out/diag4.txt | tail -30
