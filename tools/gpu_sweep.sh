#!/bin/bash
# quick per-table sweep of bench.py on one config: prints value, gemm ms, roofline frac
mkdir -p gpurun_out
CFG=${CFG:-dsv2}
for TB in ${TABLES:-mixed}; do
  timeout 300 python bench.py --config $CFG --table $TB --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${EXTRA} > gpurun_out/sw_${CFG}_${TB}.json 2> gpurun_out/sw_${CFG}_${TB}.err
  python -c "
import json,sys
try:
  d=json.load(open('gpurun_out/sw_${CFG}_${TB}.json'))
  print('${CFG} ${TB} T=%d tok/s=%.3g step=%.3fms gemm=%.3fms frac=%.3f per_expert=%.3f stages=%s' % (d['config']['tokens_per_gpu'], d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['per_expert_roofline']['frac_of_gemm'], {k: round(v,3) for k,v in d['stage_ms'].items()}))
except Exception as e: print('${CFG} ${TB} FAILED', e); print(open('gpurun_out/sw_${CFG}_${TB}.err').read()[-2000:])
"
done
