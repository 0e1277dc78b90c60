#!/bin/bash
# round measurement: GPU tests, smoke, bench on every config (default = DSV2), ncu launch list + full capture
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/final/smi.txt 2>&1
timeout 900 python bench.py --cpu-sample 128 > gpurun_out/final/bench_dsv2.json 2> gpurun_out/final/bench_dsv2.err
for c in q15 mx q2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
for c in dsv2 q15 mx q2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'route_|gather_|plan_|moe_gemm|combine_' -c 40 --csv --log-file gpurun_out/final/launches_$c.csv \
     python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/final/ncu1_$c.err
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -s 2 -c 1 -o gpurun_out/final/prof_$c -f \
     python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/final/ncu2_$c.err
done
tail -2 gpurun_out/final/pytest_gpu.log; tail -1 gpurun_out/final/smoke.log
for c in dsv2 q15 mx q2; do head -c 400 gpurun_out/final/bench_$c.json; echo; done
