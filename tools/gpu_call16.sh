mkdir -p gpurun_out
timeout 200 python tools/measure_i8_peak.py gpurun_out/i8_peak.json > gpurun_out/peaks.log 2>&1
cp gpurun_out/i8_peak.json profiles/i8_peak.json 2>/dev/null
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_moe.py tests/test_gpu_fullsize.py -k "split_k or exact or t16384" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
(time timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err) 2> gpurun_out/bench_default.time
tail -3 gpurun_out/pytest_new.log; cat gpurun_out/peaks.log gpurun_out/bench_default.time
