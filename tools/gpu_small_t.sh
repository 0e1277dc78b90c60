#!/bin/bash
# memory-bound end of the Mixtral sweep: tokens/s and HBM roofline fraction at small T
mkdir -p gpurun_out; : > gpurun_out/small_t.txt
for T in 1 4 16 64 256; do
  timeout 300 python bench.py --config mx --tokens $T --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-comparators > /tmp/b.json 2>/tmp/b.err
  echo "mx T=$T $(python -c 'import json; d=json.load(open("/tmp/b.json")); p=d["per_expert_roofline"]; print("step_ms=%.4f gemm_ms=%.4f t_roof_us=%.1f frac_gemm=%.3f alg_bytes=%.3g" % (d["ms_per_step"], d["roofline"]["kernel_ms"], p["t_roof_us"], p["frac_of_gemm"], p["alg_bytes"]))' 2>&1 | tail -1)" >> gpurun_out/small_t.txt
done
cat gpurun_out/small_t.txt
