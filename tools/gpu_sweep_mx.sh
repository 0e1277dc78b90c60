#!/bin/bash
# Mixtral token sweep (1 .. 16384) of the default bench line (mixed table chosen per T), no comparators
mkdir -p gpurun_out/sweep; : > gpurun_out/sweep/mx_sweep.txt
for T in 1 4 16 64 256 512 1024 2048 4096 8192 16384; do
  timeout 300 python bench.py --config mx --tokens $T --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > gpurun_out/sweep/mx_$T.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep/mx_$T.json')); r=d['roofline']; p=d['per_expert_roofline']; print('T=%5d tok/s=%10.0f step_ms=%.4f gemm_ms=%.4f bound=%s frac=%.3f t_roof_us=%.1f' % ($T, d['value'], d['ms_per_step'], r['kernel_ms'], r['bound'], p['frac_of_gemm'], p['t_roof_us']))" >> gpurun_out/sweep/mx_sweep.txt 2>&1
done
cat gpurun_out/sweep/mx_sweep.txt
