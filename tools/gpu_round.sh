#!/bin/bash
# one GPU session: GPU tests, smoke, bench on every BASELINE config, ncu launch list of the default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in ${CFGS:-q15 mx q2}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'route_|gather_|plan_|moe_gemm|combine_|flush' -c 200 --csv --log-file gpurun_out/launches_dsv2.csv \
     python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/ncu1.err
fi
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in gpurun_out/bench_*.json; do echo $f; head -c 600 $f; echo; done
