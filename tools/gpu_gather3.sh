#!/bin/bash
# gather occupancy variants (register pass x resident blocks): gather stage times
mkdir -p gpurun_out; O=gpurun_out/gather3; mkdir -p $O
MXM_LIB=$(pwd)/tools/variants/lib_p4b6.so timeout 900 python -m pytest tests/test_gpu_bitexact.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest p4b6 rc=$?" >> $O/pytest.log
for c in q2 q15; do
  for v in base p4b6 p4b5 p8b5 p4b4 base p4b6 p4b5; do
    LIBV=""; [ $v != base ] && LIBV=$(pwd)/tools/variants/lib_$v.so
    MXM_LIB=$LIBV timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /tmp/g.json 2>/dev/null
    echo "$c $v $(python -c 'import json; d=json.load(open("/tmp/g.json")); s=d["stage_ms"]; print("step %.4f gather %.4f plan %.4f gemm %.4f" % (d["ms_per_step"], s["gather"], s["plan"], s["gemm"]))')" >> $O/stages.txt
  done
done
tail -2 $O/pytest.log; cat $O/stages.txt
