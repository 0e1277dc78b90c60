#!/bin/bash
# 16-byte task stores in the plan: scheduler tests, plan stage A/B vs the previous build
mkdir -p gpurun_out; O=gpurun_out/${PTAG:-plan}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_moe.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in q2 q15 mx dsv2; do
  for v in ${PV:-base prev base prev}; do
    LIBV=""; [ $v != base ] && LIBV=$(pwd)/tools/variants/lib_$v.so
    MXM_LIB=$LIBV timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /tmp/g.json 2>/dev/null
    echo "$c $v $(python -c 'import json; d=json.load(open("/tmp/g.json")); s=d["stage_ms"]; print("step %.4f gather %.4f plan %.4f gemm %.4f" % (d["ms_per_step"], s["gather"], s["plan"], s["gemm"]))')" >> $O/stages.txt
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plan_kernel -c 3 --csv python bench.py --config q2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-comparators 2>/dev/null | grep gpu__time >> $O/plan_ncu.txt
tail -2 $O/pytest.log; cat $O/stages.txt; cut -c1-60,200- $O/plan_ncu.txt
