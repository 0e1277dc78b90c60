#!/bin/bash
# wait-site counters + per-stage trace of the persistent kernel for the given "cfg table T" specs
mkdir -p gpurun_out; O=gpurun_out/diag${TAG}.txt; : > $O
IFS=';' read -ra SP <<< "${SPECS}"
for spec in "${SP[@]}"; do
  set -- $spec
  echo "=== waits $spec" >> $O; timeout 300 python tools/diag_waits.py $1 $2 $3 >> $O 2>&1
  echo "=== trace $spec" >> $O; timeout 300 python tools/diag_trace.py $1 $2 $3 ${4:-} >> $O 2>&1
done
cat $O
