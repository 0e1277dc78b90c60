#!/bin/bash
mkdir -p gpurun_out/gncu
timeout 600 ncu --set full --clock-control none -k regex:gather_tok -s 2 -c 1 -o gpurun_out/gncu/g_q2 -f \
  python bench.py --config q2 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/gncu/err.txt
ncu -i gpurun_out/gncu/g_q2.ncu-rep --page details --csv > gpurun_out/gncu/details.csv 2>&1
ncu -i gpurun_out/gncu/g_q2.ncu-rep --page raw --csv > gpurun_out/gncu/raw.csv 2>&1
rm -f gpurun_out/gncu/*.ncu-rep
grep -E "Duration|DRAM Throughput|Memory Throughput|Achieved Occupancy|Warp Cycles Per Issued|Issue Slots Busy|Compute \(SM\) Throughput|L2 Hit|Stall|Registers" gpurun_out/gncu/details.csv | head -40
