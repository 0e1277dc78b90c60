set -x
mkdir -p gpurun_out
timeout 120 ./tools/probe_f8 > gpurun_out/probe_f8.txt 2>&1; echo "probe rc=$?" >> gpurun_out/probe_f8.txt
timeout 600 python bench.py --config q2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q2_base.json 2> gpurun_out/bench_q2_base.err
echo done
