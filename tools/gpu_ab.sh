#!/bin/bash
# A/B GEMM time of library variants: VARIANTS="base wait0" SPECS="q2 w4a4_g128_sym;q2 mixed" bash tools/gpu_ab.sh
mkdir -p gpurun_out; OUT=gpurun_out/ab${TAG}.txt; : > $OUT
IFS=';' read -ra SP <<< "${SPECS}"
for spec in "${SP[@]}"; do
  set -- $spec
  for v in ${VARIANTS}; do
    LIBV=""; EXTRA="MXM_AB_DUMMY=1"
    case "$v" in base) ;; env:*) EXTRA="${v#env:}" ;; *) LIBV=$(pwd)/tools/variants/lib_$v.so ;; esac
    env $EXTRA MXM_LIB=$LIBV timeout 300 python bench.py --config $1 --table ${2:-mixed} ${3:+--tokens $3} --steps ${STEPS:-5} --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /tmp/b.json 2>/tmp/b.err
    echo "$spec $v rc=$? $(python -c 'import json; d=json.load(open("/tmp/b.json")); print("gemm_ms=%.4f step_ms=%.4f pe_frac=%.3f" % (d["roofline"]["kernel_ms"], d["ms_per_step"], d["per_expert_roofline"]["frac_of_gemm"]))' 2>&1 | tail -1)" >> $OUT
  done
done
cat $OUT
