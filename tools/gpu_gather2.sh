#!/bin/bash
# gather register-pass variants: bit-exact tests (product and p8), then gather stage times
mkdir -p gpurun_out; O=gpurun_out/gather2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bitexact.py tests/test_gpu_fp8.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
MXM_LIB=$(pwd)/tools/variants/lib_p8.so timeout 900 python -m pytest tests/test_gpu_bitexact.py -q -x -p no:cacheprovider > $O/pytest_p8.log 2>&1; echo "pytest p8 rc=$?" >> $O/pytest_p8.log
for c in q15 q2 dsv2; do
  for v in base p8 p8b3 p16b2 p16b3 prev base p8; do
    LIBV=""; [ $v != base ] && LIBV=$(pwd)/tools/variants/lib_$v.so
    MXM_LIB=$LIBV timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /tmp/g.json 2>/dev/null
    echo "$c $v $(python -c 'import json; d=json.load(open("/tmp/g.json")); s=d["stage_ms"]; print("step %.4f gather %.4f gemm %.4f" % (d["ms_per_step"], s["gather"], s["gemm"]))')" >> $O/stages.txt
  done
done
tail -2 $O/pytest.log; tail -2 $O/pytest_p8.log; cat $O/stages.txt
