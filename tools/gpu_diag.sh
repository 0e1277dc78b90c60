#!/bin/bash
# wait-site breakdowns (diag build; DIAG="cfg table[;cfg table...]") + one ncu --set full capture of the GEMM
mkdir -p gpurun_out; OUT=gpurun_out/diag${TAG}.txt; : > $OUT
IFS=';' read -ra SPECS <<< "${DIAG}"
for spec in "${SPECS[@]}"; do
  [ -n "$spec" ] && timeout 300 python tools/diag_waits.py $spec >> $OUT 2>&1
done
if [ -n "$NCUCFG" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -s 1 -c 1 -o gpurun_out/prof_${NCUCFG}${TAG} -f \
     python bench.py --config $NCUCFG ${NCUARGS} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/ncu${TAG}.err
  echo "ncu rc=$?" >> $OUT
fi
cat $OUT
