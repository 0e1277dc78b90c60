timeout 900 python -m pytest tests/test_gpu_bitexact.py tests/test_gpu_moe.py -q -x -p no:cacheprovider 2>&1 | tail -2
VARIANTS="base" SPECS="q2 w4a4_g128_sym;q2 mixed;q2 w8a8_g-1_sym;dsv2 mixed;q15 mixed;mx mixed;mx mixed 1" bash tools/gpu_ab.sh
TRACE_PRODUCER=1 MXM_LIB=$(pwd)/tools/variants/lib_trace_prod.so timeout 300 python tools/diag_trace.py q2 w4a4_g128_sym > gpurun_out/trace_g128_split.txt 2>&1; tail -n 4 gpurun_out/trace_g128_split.txt
