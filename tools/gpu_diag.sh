#!/bin/bash
# diagnostics: mixtral crash isolation + wait-site breakdowns
mkdir -p gpurun_out
: > gpurun_out/diag_mx.txt
for tb in w4a16_g128_asym w8a8_g-1_sym mixed; do
  for T in 64 512; do
    timeout 120 python bench.py --config mx --tokens $T --table $tb --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-comparators > /tmp/o.json 2>/tmp/o.err
    echo "mx $tb T=$T rc=$? $(head -c 300 /tmp/o.json) $(grep -m1 -i error /tmp/o.err)" >> gpurun_out/diag_mx.txt
  done
done
: > gpurun_out/diag_waits.txt
for a in "dsv2 mixed" "q15 mixed" "q15 w8a8_g-1_sym" "q2 mixed" "q2 w8a8_g-1_sym" "q2 w4a4_g128_sym"; do
  timeout 300 python tools/diag_waits.py $a >> gpurun_out/diag_waits.txt 2>&1
done
cat gpurun_out/diag_mx.txt gpurun_out/diag_waits.txt
