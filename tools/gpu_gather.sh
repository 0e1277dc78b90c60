#!/bin/bash
# token-major gather with lane-parallel g128 divisions: bit-exact tests, then per-stage times vs the previous build
mkdir -p gpurun_out; O=gpurun_out/gather; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bitexact.py tests/test_gpu_fp8.py tests/test_gpu_moe.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in q15 q2 mx; do
  for v in base prev base prev; do
    LIBV=""; [ $v != base ] && LIBV=$(pwd)/tools/variants/lib_$v.so
    MXM_LIB=$LIBV timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /tmp/g.json 2>/dev/null
    echo "$c $v $(python -c 'import json; d=json.load(open("/tmp/g.json")); s=d["stage_ms"]; print("step %.4f gather %.4f gemm %.4f" % (d["ms_per_step"], s["gather"], s["gemm"]))')" >> $O/stages.txt
  done
done
tail -2 $O/pytest.log; cat $O/stages.txt
