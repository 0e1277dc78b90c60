#!/bin/bash
# lagged expert interleave of the queue (plan.cu MXM_INTERLEAVE_LAG variants): parity through a variant, GEMM A/B
mkdir -p gpurun_out; O=gpurun_out/lag; mkdir -p $O
MXM_LIB=$(pwd)/tools/variants/lib_lag8.so timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_bitexact.py -q -x -p no:cacheprovider > $O/pytest_lag8.log 2>&1; echo "pytest lag8 rc=$?" >> $O/pytest_lag8.log
NOTEST=1 VARIANTS="base lag4 lag8 lag16" SPECS="q2 mixed;q15 mixed;dsv2 mixed;mx mixed" TAG=20 bash tools/gpu_ab2.sh > /dev/null 2>&1
cp gpurun_out/ab20.txt $O/
for v in base lag8; do
  LIBV=""; [ $v != base ] && LIBV=$(pwd)/tools/variants/lib_$v.so
  MXM_LIB=$LIBV timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:moe_gemm -s 2 -c 1 --csv \
    python bench.py --config q2 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/$v /" | awk -F'","' '{print $1, $(NF-2), $NF}' >> $O/dram.txt
done
tail -2 $O/pytest_lag8.log; cat $O/ab20.txt; cat $O/dram.txt
