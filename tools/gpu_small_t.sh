#!/bin/bash
# Mixtral small-T step times (device time per block step, mixed table), several repeats
mkdir -p gpurun_out; : > gpurun_out/small_t${TAG}.txt
for T in 1 4 16 64; do
  for rep in 1 2; do
    timeout 300 python bench.py --config mx --tokens $T --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-comparators > /tmp/s.json 2>/dev/null
    python -c "import json; d=json.load(open('/tmp/s.json')); print('T=%d step_ms=%.4f gemm_ms=%.4f stages=%s' % ($T, d['ms_per_step'], d['roofline']['kernel_ms'], {k: round(v, 4) for k, v in d['stage_ms'].items()}))" >> gpurun_out/small_t${TAG}.txt
  done
done
cat gpurun_out/small_t${TAG}.txt
