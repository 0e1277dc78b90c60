#!/bin/bash
# wait-site counters and per-stage trace with and without the epilogue's work (g128 structure analysis)
mkdir -p gpurun_out; O=gpurun_out/diag_epi.txt; : > $O
for v in diag diagepi; do echo "=== waits $v q2 w4a4_g128" >> $O; MXM_LIB=$(pwd)/tools/variants/lib_$v.so timeout 300 python tools/diag_waits.py q2 w4a4_g128_sym 16384 >> $O 2>&1; done
for v in diag diagepi; do echo "=== waits $v q2 w4a4_pc" >> $O; MXM_LIB=$(pwd)/tools/variants/lib_$v.so timeout 300 python tools/diag_waits.py q2 w4a4_g-1_sym 16384 >> $O 2>&1; done
for v in trace traceepi; do echo "=== trace $v q2 w4a4_g128" >> $O; MXM_LIB=$(pwd)/tools/variants/lib_$v.so timeout 300 python tools/diag_trace.py q2 w4a4_g128_sym 16384 full >> $O 2>&1; done
cat $O
