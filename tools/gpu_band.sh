#!/bin/bash
# banded n-tile-major emission of large experts (plan.cu MXM_BAND_MB): scheduler tests, GEMM A/B, DRAM bytes
mkdir -p gpurun_out; O=gpurun_out/band; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_moe.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
NOTEST=1 VARIANTS="base noband band8 band32" SPECS="q2 mixed;q15 mixed;dsv2 mixed;q2 w8a8_g-1_sym" TAG=17 bash tools/gpu_ab2.sh > /dev/null 2>&1
cp gpurun_out/ab17.txt $O/
for v in base noband; do
  LIBV=""; [ $v != base ] && LIBV=$(pwd)/tools/variants/lib_$v.so
  for c in q2 q15; do
    MXM_LIB=$LIBV timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:moe_gemm -s 2 -c 1 --csv \
      python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators 2>/dev/null | grep -E "dram__|lts__|gpu__time" | sed "s/^/$v $c /" >> $O/dram.txt
  done
done
tail -2 $O/pytest.log; cat $O/ab17.txt; cat $O/dram.txt
