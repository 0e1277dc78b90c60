#!/bin/bash
# one GPU session: i8 peak, smoke, bench (default workload), ncu launch list + full capture of the GEMM
mkdir -p gpurun_out
CFG=${CFG:-dsv2}
timeout 120 python tools/measure_i8_peak.py gpurun_out/i8_peak.json > gpurun_out/i8.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config $CFG ${BENCH_ARGS} > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench rc=$?"
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'route_|gather_|plan_|moe_gemm|combine_' -c 40 --csv --log-file gpurun_out/launches_$CFG.csv \
     python bench.py --config $CFG --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/ncu1.err
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -s 1 -c 1 -o gpurun_out/prof_$CFG -f \
     python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>gpurun_out/ncu2.err
fi
cat gpurun_out/i8.log gpurun_out/smoke.log; tail -3 gpurun_out/bench_$CFG.err; cat gpurun_out/bench_$CFG.json
