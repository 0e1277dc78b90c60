#!/bin/bash
mkdir -p gpurun_out/pncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plan_kernel -s 2 -c 1 -o gpurun_out/pncu/p_q2 -f \
  python bench.py --config q2 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/pncu/err.txt
ncu -i gpurun_out/pncu/p_q2.ncu-rep --page details --csv > gpurun_out/pncu/details.csv 2>&1
ncu -i gpurun_out/pncu/p_q2.ncu-rep --page source --csv --print-source sass > gpurun_out/pncu/source.csv 2>&1
ncu -i gpurun_out/pncu/p_q2.ncu-rep --page source --csv --print-source cuda > gpurun_out/pncu/source_cuda.csv 2>&1
rm -f gpurun_out/pncu/*.ncu-rep
ls -la gpurun_out/pncu
