#!/bin/bash
# per-task timeline of CTA 0 + per-CTA finish spread (tools/diag_tasks.py, -DMXM_TRACE_TASKS build)
mkdir -p gpurun_out; O=gpurun_out/diag_tasks.txt; : > $O
for spec in "q2 w4a4_g128_sym 16384" "q2 w4a4_g-1_sym 16384" "q2 mixed 16384" "dsv2 mixed 4096" "q15 mixed 8192"; do
  echo "=== $spec" >> $O; timeout 300 python tools/diag_tasks.py $spec >> $O 2>&1
done
cat $O
