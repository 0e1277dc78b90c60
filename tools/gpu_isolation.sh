#!/bin/bash
# isolation runs (tools/isolation.py) under ncu: per-launch time, DRAM bytes / throughput, tensor-pipe activity
mkdir -p gpurun_out
timeout 900 ncu --clock-control none -k regex:moe_gemm \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/isolation_ncu${TAG}.csv python tools/isolation.py --reps 1 > gpurun_out/isolation_ncu_stdout${TAG}.txt 2>&1
echo "ncu rc=$?"
