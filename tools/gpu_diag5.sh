#!/bin/bash
mkdir -p gpurun_out
MXM_LIB=$(pwd)/tools/variants/lib_nan2.so NANTEST2=1 timeout 200 python tools/diag_mix.py 8 2048 14336 512 2 wa8,wo4,wo4,wo4 > gpurun_out/diag5.txt 2>&1
MXM_LIB=$(pwd)/tools/variants/lib_nan2.so NANTEST2=1 timeout 200 python tools/diag_mix.py 8 2048 14336 512 2 wa8,wo4 >> gpurun_out/diag5.txt 2>&1
grep -v CUDAEvent gpurun_out/diag5.txt | tail -30
