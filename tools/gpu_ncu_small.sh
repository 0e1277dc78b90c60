#!/bin/bash
# full ncu capture of the group-GEMM at a memory-bound Mixtral point (VERDICT r1 item 4 evidence)
mkdir -p gpurun_out/ncu_small
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -s 3 -c 1 \
  -o gpurun_out/ncu_small/prof_mx_T${T:-8} -f python bench.py --config mx --tokens ${T:-8} --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2> gpurun_out/ncu_small/ncu.err
echo "rc=$?"
