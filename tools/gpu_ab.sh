#!/bin/bash
# A/B timing of library variants: VARIANTS="tools/variants/lib_x.so ..." (empty entry = product lib),
# TABLES="mixed w16 ...", CFG=dsv2. One bench line per (variant, table) in gpurun_out/ab.txt
mkdir -p gpurun_out
CFG=${CFG:-dsv2}
for v in default ${VARIANTS}; do
  for tb in ${TABLES:-mixed}; do
    if [ "$v" = default ]; then unset MXM_LIB; else export MXM_LIB=$(pwd)/$v; fi
    out=$(timeout 300 python bench.py --config $CFG --table $tb --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e --no-comparators ${EXTRA} 2>gpurun_out/ab_err.txt)
    echo "$v $tb $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("step_ms=%.4f gemm_ms=%.4f frac=%.3f" % (d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"]))' 2>&1 | tail -1)" | tee -a gpurun_out/ab.txt
  done
done
