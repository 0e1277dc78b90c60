#!/bin/bash
# GEMM time of one config under several uniform tables: CFG=q2 TABLES="w4a4_g128_sym ..." bash tools/gpu_tables.sh
mkdir -p gpurun_out; OUT=gpurun_out/tables${TAG}.txt; : > $OUT
for tb in ${TABLES}; do
  timeout 400 python bench.py --config ${CFG:-q2} --table $tb --steps ${STEPS:-5} --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /tmp/b.json 2>/tmp/b.err
  echo "${CFG:-q2} $tb rc=$? $(python -c '
import json,sys; d=json.load(open(sys.argv[1])); p=d["per_expert_roofline"]
print("step_ms=%.4f gemm_ms=%.4f frac=%.3f t_roof_us=%.0f" % (d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"], p["t_roof_us"]))' /tmp/b.json 2>&1 | tail -1)" >> $OUT
done
IFS=';' read -ra SPECS <<< "${DIAG}"
for spec in "${SPECS[@]}"; do
  [ -n "$spec" ] && timeout 300 python tools/diag_waits.py $spec >> $OUT 2>&1
done
cat $OUT
