#!/bin/bash
# round-2 measurement session: GPU tests, smoke, bench (default = Q2 headline) + other configs,
# ncu launch list of the default bench and one full capture of the group-GEMM kernel
O=gpurun_out/${TAG:-r02}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench_q2.json 2> $O/bench_q2.err
for c in ${CFGS:-dsv2 q15 mx}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'route_|gather_|plan_|moe_gemm|combine_' -c 40 --csv --log-file $O/launches_q2.csv \
     python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>$O/ncu1.err
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -s 2 -c 1 -o $O/prof_q2 -f \
     python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>$O/ncu2.err
  for c in ${NCU_CFGS:-}; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'route_|gather_|plan_|moe_gemm|combine_' -c 40 --csv --log-file $O/launches_$c.csv \
       python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>$O/ncu1_$c.err
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -s 2 -c 1 -o $O/prof_$c -f \
       python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>$O/ncu2_$c.err
  done
fi
if [ -n "$NCU" ]; then
  # summaries only travel back (gpurun_out is capped at 64 MiB): key counters + launch shares per config and the
  # traffic json tagged with this library's sha, then the raw reports are dropped
  python tools/summarize_profiles.py $O $O/summ > $O/summ.log 2>&1
  rm -f $O/*.ncu-rep
fi
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log
for f in $O/bench_*.json; do echo $f; head -c 300 $f; echo; done
