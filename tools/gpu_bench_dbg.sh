#!/bin/bash
# bench runs with an interrupt-on-timeout (a Python traceback shows where a hang sits)
mkdir -p gpurun_out/dbg
for c in ${CFGS:-q2 q15}; do
  timeout -s INT ${BT:-240} python -X faulthandler bench.py --config $c ${EXTRA:-} > gpurun_out/dbg/bench_$c.json 2> gpurun_out/dbg/bench_$c.err
  echo "$c rc=$?" >> gpurun_out/dbg/rc.txt
done
cat gpurun_out/dbg/rc.txt; for c in ${CFGS:-q2 q15}; do tail -25 gpurun_out/dbg/bench_$c.err; head -c 300 gpurun_out/dbg/bench_$c.json; echo; done
